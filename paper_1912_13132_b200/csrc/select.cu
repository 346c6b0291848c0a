// select.cu -- the grid-search consumer of the CV losses (PAPER.md
// §4.3.3): the global choice zeta_hat_CV = argmin_c C~V(zeta_c), global
// RMSPEs sqrt(C~V / n_V), local RMSPEs per subset, and each subset's locally best
// configuration with the number of subsets every configuration wins (the dot sizes of the
// paper's Fig. "fit").  Operates on the device-resident per-subset
// losses of the last evaluation; deterministic (fixed scan orders, ties -> lowest c).
#include <cmath>
#include <cstdint>

#include "pgpcv_internal.h"

namespace pgpcv {
namespace {

// One thread per subset s: local RMSPE sqrt(z_{s,c} / m_s) for every config and the
// locally best config argmin_c z_{s,c} (failed configs skipped; -1 when m_s = 0 or all
// failed).  wins[c] counts the subsets whose local best is c.
__global__ void select_local_kernel(const double *subset_loss, const uint8_t *fail, const int64_t *val_off,
                                    int64_t N, int32_t C, double *local_rmspe, int32_t *local_best,
                                    int32_t *wins) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= N) return;
    const int64_t m = val_off[s + 1] - val_off[s];
    const double qnan = __longlong_as_double(0x7ff8000000000000ll);
    int32_t best = -1;
    double bl = 0.0;
    for (int32_t c = 0; c < C; ++c) {
        const double z = subset_loss[s * C + c];
        const bool ok = m > 0 && !fail[s * C + c];
        local_rmspe[s * C + c] = ok ? sqrt(z / (double)m) : qnan;
        if (ok && (best < 0 || z < bl)) {
            best = c;
            bl = z;
        }
    }
    local_best[s] = best;
    if (best >= 0) atomicAdd(wins + best, 1);
}

// One CTA: global RMSPE per config and the global argmin (written to best_out).
__global__ void select_global_kernel(const double *loss, int32_t C, int64_t n_val, double *rmspe,
                                     int32_t *best_out) {
    for (int c = threadIdx.x; c < C; c += blockDim.x) rmspe[c] = sqrt(loss[c] / (double)n_val);
    if (threadIdx.x == 0) {
        int32_t best = -1;
        double bl = 0.0;
        for (int32_t c = 0; c < C; ++c) {
            const double l = loss[c];
            if (l == l && (best < 0 || l < bl)) {  // NaN (failed config) never wins
                best = c;
                bl = l;
            }
        }
        *best_out = best;
    }
}

}  // namespace

cudaError_t launch_select(const double *subset_loss, const uint8_t *fail, const int64_t *val_off,
                          const double *loss, int64_t N, int32_t C, int64_t n_val, double *rmspe,
                          double *local_rmspe, int32_t *best, int32_t *wins, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(wins, 0, sizeof(int32_t) * C, st);
    if (e != cudaSuccess) return e;
    if (N > 0)
        select_local_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(subset_loss, fail, val_off, N, C,
                                                                         local_rmspe, best, wins);
    select_global_kernel<<<1, 256, 0, st>>>(loss, C, n_val, rmspe, best + N);
    return cudaGetLastError();
}

}  // namespace pgpcv
