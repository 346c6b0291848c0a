// cv_small.cu -- the per-(subset, config) evaluation of cv_kernel.cu for SMALL subsets
// (k <= kSmallK), one WARP per item.
//
// Same mathematics (Eq.3/Eq.4 per subset; Eq.2 for -2 log L): A =
// Sigma(theta) + lambda I generated from the staged coordinates, FP64 Cholesky with y_T as
// a bordered row, backward substitution, prediction, SSPE.  What changes is the shape of
// the parallelism.  At k ~ 350 (BASELINE configs c2, c3) a subset's update is too short to
// hide the serial pivot chain of its diagonal blocks when a whole CTA works on one subset
// (cv_kernel.cu spends 36 % of its time in that chain at c3).  Here every warp owns one item
// and 16 items are in flight per SM, so one item's pivot chain overlaps fifteen other
// items' DMMA updates.
//
// Per warp, for 8-wide block columns j (columns j0..j0+7), rows j0..k in groups of 64:
//   acc   = -A[group rows, j0:j0+8]              generated in registers (2 entries/lane/tile)
//   acc  += L[group rows, 0:j0] . L[j0:j0+8, 0:j0]^T     DMMA m8n8k4, operands from global
//           memory through L1 (the 8-row B fragment is reused by the group's 8 tiles)
//   diagonal tile: 8 pivots by lanes 0..7 (register shuffles, rsqrt), then the 8 x 8
//           inverse by columns (lanes 0..7 in parallel) -- in per-warp SMEM
//   other tiles: X = C . Linv^T (2 DMMA per tile, A fragments shuffled out of acc)
// The factor is column-major with ld = roundup(k+1, 8) (row k: z = L^{-1} y_T); each
// block's inverse is kept for the back-substitution (alpha_j = Linv_j^T t_j).  alpha lives
// in per-warp SMEM.  GLS items (kCvGls) always go to cv_kernel.cu.
#include <algorithm>
#include <cmath>
#include <cstdint>

#include "pgpcv_internal.h"
#include "pgpcv_device.cuh"

namespace pgpcv {
namespace {

constexpr int WPB = 8;           // warps (items) per CTA
constexpr int TPB = WPB * 32;
constexpr int KS = kSmallK;      // largest k handled here
constexpr int GR = 8;            // row tiles of 8 rows per update group (64 rows)
constexpr int DS = 9;            // row stride of the per-warp 8 x 8 scratch blocks
constexpr int WS_DBL = KS + 2 * 8 * DS + 8;  // alpha, L_jj, Linv_jj, reciprocal pivots
constexpr size_t SMEM_BYTES = sizeof(double) * (EXP_TAB + (size_t)WPB * WS_DBL);
static_assert(SMEM_BYTES <= 110 * 1024, "two CTAs per SM");

__host__ __device__ __forceinline__ int64_t small_ld(int64_t k) { return ((k + 1 + 7) / 8) * 8; }

__global__ void __launch_bounds__(TPB, 2) cv_small_kernel(CvArgs a) {
    extern __shared__ __align__(16) double smem[];
    double *etab = smem;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    if (tid < EXP_TAB) etab[tid] = kExp2Tab[tid];
    __syncthreads();
    double *ws = smem + EXP_TAB + warp * WS_DBL;
    double *alpha = ws;            // [KS]
    double *Ls = ws + KS;          // L_jj   [8][DS]
    double *Li = Ls + 8 * DS;      // Linv_jj [8][DS]
    double *rdg = Li + 8 * DS;     // 1 / L_jj[i][i]
    const int gw = blockIdx.x * WPB + warp;
    double *L = a.work + (size_t)gw * a.slot_stride;

    for (;;) {
        int item = 0;
        if (lane == 0) item = (int)atomicAdd(reinterpret_cast<unsigned int *>(a.counter), 1u);
        item = __shfl_sync(0xffffffffu, item, 0);
        if (item >= a.n_items) break;
        const int s = a.items[item].x, c = a.items[item].y;
        const int64_t toff = a.train_off[s];
        const int k = (int)(a.train_off[s + 1] - toff);
        const int64_t voff = a.val_off[s];
        const int m = (int)(a.val_off[s + 1] - voff);
        const double *tx = a.tx + toff, *ty = a.ty + toff, *tv = a.tv + toff;
        const double range = a.params[3 * c], sigma2 = a.params[3 * c + 1];
        const double lam = a.params[3 * c + 2] / sigma2;
        const double ninv = -1.0 / range;
        const int64_t oi = (int64_t)s * a.out_C + (a.out_C > 1 ? c : 0);
        const int ld = (int)small_ld(k);
        double *linvG = L + (size_t)ld * k;  // inverse of every 8 x 8 diagonal block
        const int nb = (k + 7) / 8;
        bool failed = false;
        double logdet = 0.0;

        // ---------------- blocked left-looking Cholesky, bordered y_T row ----------------
        for (int jb = 0; jb < nb && !failed; ++jb) {
            const int j0 = jb * 8, jw = min(8, k - j0);
            double cxv[2], cyv[2], cvv[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int cc = j0 + 2 * t + e;
                const bool ok = cc < k;
                cxv[e] = ok ? __ldg(tx + cc) : 0.0;
                cyv[e] = ok ? __ldg(ty + cc) : 0.0;
                cvv[e] = ok ? __ldg(tv + cc) : 0.0;
            }
            const bool bvalid = j0 + g < k;  // this lane's row of the B fragment exists
            for (int r0 = j0; r0 <= k; r0 += 8 * GR) {
                double acc[GR][2];
#pragma unroll
                for (int q = 0; q < GR; ++q) {
                    const int r = r0 + 8 * q + g;
                    const double rx = r < k ? __ldg(tx + r) : 0.0, ry = r < k ? __ldg(ty + r) : 0.0;
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int cc = j0 + 2 * t + e;
                        const double dx = rx - cxv[e], dy = ry - cyv[e];
                        double v = -exp_neg(sqrt(dx * dx + dy * dy) * ninv, etab);
                        v = r == cc ? -(1.0 + lam) : v;               // exp(0) + lambda
                        v = r == k ? -cvv[e] : v;                     // bordered y_T
                        v = (cc >= k || r > k || r < cc) ? 0.0 : v;   // pad / upper
                        acc[q][e] = v;
                    }
                }
                // acc += L[rows, 0:j0] . L[j0:j0+8, 0:j0]^T
                for (int kk = 0; kk < j0; kk += 4) {
                    const double *col = L + (size_t)(kk + t) * ld;
                    const double b = bvalid ? col[j0 + g] : 0.0;
#pragma unroll
                    for (int q = 0; q < GR; ++q) {
                        if (r0 + 8 * q > k) break;  // warp-uniform
                        const int r = r0 + 8 * q + g;
                        const double av = r <= k ? col[r] : 0.0;
                        dmma(acc[q], av, b);
                    }
                }
                // columns past the matrix stay exactly 0 (their Linv entries are 0 too)
#pragma unroll
                for (int q = 0; q < GR; ++q)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        if (j0 + 2 * t + e >= k) acc[q][e] = 0.0;

                if (r0 == j0) {
                    // ---- diagonal tile: C = -acc[0], 8 pivots, inverse ----
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int n = 2 * t + e;
                        Ls[g * DS + n] = n <= g ? -acc[0][e] : 0.0;
                    }
                    __syncwarp();
                    double va[8];
#pragma unroll
                    for (int c2 = 0; c2 < 8; ++c2) va[c2] = (lane < 8) ? Ls[lane * DS + c2] : 0.0;
                    bool bad = false;
#pragma unroll
                    for (int c2 = 0; c2 < 8; ++c2) {
                        if (c2 < jw && !bad) {
                            const double piv = __shfl_sync(0xffffffffu, va[c2], c2);
                            double lu[8];
#pragma unroll
                            for (int c3 = c2 + 1; c3 < 8; ++c3) lu[c3] = __shfl_sync(0xffffffffu, va[c2], c3);
                            if (!(piv > 0.0)) {  // not positive definite (R12); warp-uniform
                                bad = true;
                            } else {
                                const double inv = rsqrt(piv);
                                const double rp = inv * inv;
#pragma unroll
                                for (int c3 = c2 + 1; c3 < 8; ++c3) va[c3] -= va[c2] * (lu[c3] * rp);
                                va[c2] = lane == c2 ? piv * inv : (lane > c2 ? va[c2] * inv : va[c2]);
                                if (lane == c2) rdg[c2] = inv;
                            }
                        }
                    }
                    if (bad) {
                        failed = true;
                        break;
                    }
                    // in the last block (jw < 8) the bordered row k = j0 + jw lies inside the
                    // diagonal tile: its pivot-loop values are z = L^{-1} y_T for the block
                    if (jw < 8 && lane == jw) {
#pragma unroll
                        for (int c2 = 0; c2 < 8; ++c2)
                            if (c2 < jw) L[(size_t)(j0 + c2) * ld + k] = va[c2];
                    }
                    if (lane < 8) {
#pragma unroll
                        for (int c2 = 0; c2 < 8; ++c2) Ls[lane * DS + c2] = (c2 <= lane && lane < jw) ? va[c2] : 0.0;
                    }
                    __syncwarp();
                    // Linv column n (lane n < jw): x_r = ((r == n) - sum_{p<r} L[r][p] x_p) / L[r][r]
                    if (lane < 8) {
                        double x[8];
#pragma unroll
                        for (int r = 0; r < 8; ++r) {
                            double v = (r == lane) ? 1.0 : 0.0;
#pragma unroll
                            for (int p = 0; p < r; ++p) v -= Ls[r * DS + p] * x[p];
                            x[r] = (r < lane || r >= jw || lane >= jw) ? 0.0 : v * rdg[r];
                        }
#pragma unroll
                        for (int r = 0; r < 8; ++r) Li[r * DS + lane] = x[r];
                    }
                    __syncwarp();
                    // L_jj and Linv_jj to the slot; log det for -2 log L
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int n = 2 * t + e;
                        if (n <= g && g < jw) L[(size_t)(j0 + n) * ld + j0 + g] = Ls[g * DS + n];
                        linvG[(size_t)jb * 64 + g * 8 + n] = Li[g * DS + n];
                    }
                    if (a.flags & kCvNll) logdet += warp_sum(lane < jw ? log(Ls[lane * DS + lane]) : 0.0);
                }
                // ---- X = C . Linv^T for the group's tiles (the diagonal tile excepted) ----
#pragma unroll
                for (int q = 0; q < GR; ++q) {
                    if (r0 + 8 * q > k) break;          // warp-uniform
                    if (r0 == j0 && q == 0) continue;   // L_jj itself
                    double xo[2] = {0.0, 0.0};
#pragma unroll
                    for (int sl = 0; sl < 2; ++sl) {
                        const int src = 4 * g + 2 * sl + (t >> 1);
                        const double v0 = __shfl_sync(0xffffffffu, acc[q][0], src);
                        const double v1 = __shfl_sync(0xffffffffu, acc[q][1], src);
                        dmma(xo, (t & 1) ? v1 : v0, Li[g * DS + 4 * sl + t]);
                    }
                    const int r = r0 + 8 * q + g;
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int cc = j0 + 2 * t + e;
                        if (cc < j0 + jw && r <= k) L[(size_t)cc * ld + r] = -xo[e];
                    }
                }
                __syncwarp();
            }
            __syncwarp();  // this column's stores before the next column's loads (same warp)
        }

        if (failed) {
            if (lane == 0) {
                const double qnan = __longlong_as_double(0x7ff8000000000000ll);
                if (a.flags & kCvPredict) a.subset_loss[oi] = qnan;
                if (a.flags & kCvNll) a.subset_nll[oi] = qnan;
                a.fail[oi] = 1;
            }
            continue;
        }
        if (a.flags & kCvNll) {  // Eq.2 from the same factor (see cv_kernel.cu)
            double zz = 0.0;
            for (int cc = lane; cc < k; cc += 32) {
                const double zc = L[(size_t)cc * ld + k];
                zz += zc * zc;
            }
            zz = warp_sum(zz);
            if (lane == 0) {
                const double kd = (double)k;
                a.subset_nll[oi] = kd * log(2.0 * 3.14159265358979323846) + kd * log(sigma2) + 2.0 * logdet +
                                   zz / sigma2;
            }
        }
        if (!(a.flags & kCvPredict) || m == 0) {
            if (lane == 0) {
                if (a.flags & kCvPredict) a.subset_loss[oi] = 0.0;
                a.fail[oi] = 0;
            }
            continue;
        }

        // ---------------- backward substitution L^T alpha = z ----------------
        for (int jb = nb - 1; jb >= 0; --jb) {
            const int j0 = jb * 8, jw = min(8, k - j0), rs = j0 + jw;
            double p[8];
#pragma unroll
            for (int cI = 0; cI < 8; ++cI) p[cI] = 0.0;
            for (int r = rs + lane; r < k; r += 32) {
                const double ar = alpha[r];
#pragma unroll
                for (int cI = 0; cI < 8; ++cI)
                    if (cI < jw) p[cI] += L[(size_t)(j0 + cI) * ld + r] * ar;
            }
            double tl = 0.0;  // t_lane = z_{j0+lane} - L[rs:, j0+lane] . alpha[rs:]
#pragma unroll
            for (int cI = 0; cI < 8; ++cI) {
                const double tot = warp_sum(p[cI]);
                if (lane == cI) tl = tot;
            }
            tl = lane < jw ? L[(size_t)(j0 + lane) * ld + k] - tl : 0.0;
            double al = 0.0;  // alpha_j = Linv_j^T t_j
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const double tr = __shfl_sync(0xffffffffu, tl, r);
                if (lane < jw && r >= lane && r < jw) al += linvG[(size_t)jb * 64 + r * 8 + lane] * tr;
            }
            if (lane < jw) alpha[j0 + lane] = al;
            __syncwarp();
        }

        // ---------------- prediction and squared error (Eq.3, Eq.4) ----------------
        const double *vx = a.vx + voff, *vy = a.vy + voff, *vv = a.vv + voff;
        double loss = 0.0;
        for (int v = 0; v < m; ++v) {
            const double px = __ldg(vx + v), py = __ldg(vy + v);
            double sum = 0.0;
            for (int j = lane; j < k; j += 32) {
                const double dx = px - __ldg(tx + j), dy = py - __ldg(ty + j);
                sum += exp_neg(sqrt(dx * dx + dy * dy) * ninv, etab) * alpha[j];
            }
            sum = warp_sum(sum);
            if (a.yhat && lane == 0) a.yhat[voff + v] = sum;
            const double e = sum - __ldg(vv + v);
            loss += e * e;
        }
        if (lane == 0) {
            a.subset_loss[oi] = loss;
            a.fail[oi] = 0;
        }
        __syncwarp();
    }
}

}  // namespace

size_t cv_small_slot_doubles(int64_t kmax) {
    // column-major (k+1) x k factor + the 8 x 8 inverses + slack, 256-B aligned
    const int64_t k = std::max<int64_t>(kmax, 1);
    const size_t d = (size_t)small_ld(k) * k + (size_t)((k + 7) / 8) * 64 + 64;
    return (d + 31) / 32 * 32;
}

int cv_small_warps_per_cta() { return WPB; }

cudaError_t cv_small_occupancy(int *blocks_per_sm) {
    cudaError_t e = cudaFuncSetAttribute(cv_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)SMEM_BYTES);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, cv_small_kernel, TPB, SMEM_BYTES);
}

cudaError_t launch_cv_small(const CvArgs &a, int grid, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(cv_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)SMEM_BYTES);
    if (e != cudaSuccess) return e;
    cv_small_kernel<<<grid, TPB, SMEM_BYTES, st>>>(a);
    return cudaGetLastError();
}

}  // namespace pgpcv
