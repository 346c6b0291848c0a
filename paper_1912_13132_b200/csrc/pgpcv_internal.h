// pgpcv_internal.h -- declarations shared by the libpgpcv translation units (not part of
// the ABI; never included by anything outside csrc/).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace pgpcv {

// ----------------------------------------------------------------------------------------
// Batched CV kernel (Eq.3/Eq.4 per (subset, config)).
// ----------------------------------------------------------------------------------------
struct CvArgs {
    const int64_t *train_off;   // [N+1] CSR offsets into the staged training arrays
    const int64_t *val_off;     // [N+1] CSR offsets of the prediction targets (validation
                                //       points for evaluate, test points for predict)
    const double *tx, *ty, *tv; // staged training coordinates / values (subset-contiguous)
    const double *vx, *vy, *vv; // staged target coordinates / values
    const double *params;       // [C*3] (range, sigma2, nugget)
    int32_t C;
    const int2 *items;          // [n_items] (subset, config), LPT order
    int32_t n_items;
    unsigned int *counter;      // dynamic work counter (zeroed before launch)
    double *work;               // n_slots * slot_stride doubles: one factor per resident CTA
    size_t slot_stride;
    int32_t out_C;              // output row stride: entry (s, c) at s*out_C + (out_C > 1 ? c : 0)
    int32_t flags;              // kCvPredict | kCvNll
    double *subset_loss;        // [N*out_C] SSPE of the targets (kCvPredict)
    double *subset_nll;         // [N*out_C] -2 log-likelihood of the training data (kCvNll)
    double *yhat;               // [sum of targets] kriging predictions, or nullptr
    uint8_t *fail;              // [N*out_C] 1 = not positive definite
};
constexpr int32_t kCvPredict = 1;  // back-substitution, prediction, SSPE (Eq.3, Eq.4)
constexpr int32_t kCvNll = 2;      // -2 log-likelihood from the same factor (Eq.2)

// Kernel geometry (see cv_kernel.cu for the derivation).
constexpr int kMT = 128;        // rows per row tile
constexpr int kNB = 64;         // block-column width of the left-looking Cholesky
constexpr int kThreads = 256;   // 8 warps
size_t cv_kernel_smem_bytes();
int cv_kernel_max_k();
size_t cv_kernel_slot_doubles(int64_t kmax);  // factor + back-substitution scratch
// leading dimension (doubles) of a k-point factor: column-major (k+1) x k, +1 bordered row
__host__ __device__ inline int64_t factor_ld(int64_t k) { return ((k + 1 + 15) / 16) * 16; }

cudaError_t launch_cv_kernel(const CvArgs &a, int grid, cudaStream_t st);
cudaError_t cv_kernel_occupancy(int *blocks_per_sm);
// out[c] = sum_s vals[s*C + c] over subsets s with mask_off[s+1] > mask_off[s] (all subsets
// when mask_off is null), in ascending s; NaN (and status[c] = first failing s) on failure.
cudaError_t launch_reduce(const double *vals, const uint8_t *fail, const int64_t *mask_off, int64_t N,
                          int32_t C, double *out, int32_t *status, cudaStream_t st);

// Grid-search consumer (select.cu): best[0..N-1] local argmin per subset, best[N] global.
cudaError_t launch_select(const double *subset_loss, const uint8_t *fail, const int64_t *val_off,
                          const double *loss, int64_t N, int32_t C, int64_t n_val, double *rmspe,
                          double *local_rmspe, int32_t *best, int32_t *wins, cudaStream_t st);

// ----------------------------------------------------------------------------------------
// Partition kernels (Alg.1 lines 2-3).
// ----------------------------------------------------------------------------------------
struct Axis {
    const double *e;   // [K+1] tile edges
    const double *lo;  // [K]   e_i - delta
    const double *hi;  // [K]   e_{i+1} + delta, hi[K-1] = +inf
    int32_t K;
};

cudaError_t launch_validate(int64_t n, const double *x, const double *y, const double *v,
                            const uint8_t *role, double xmin, double xmax, double ymin,
                            double ymax, unsigned long long *stats, cudaStream_t st);
cudaError_t launch_count(int64_t n, const double *x, const double *y, const uint8_t *role,
                         Axis ax, Axis ay, unsigned int *train_cnt, unsigned int *val_cnt,
                         unsigned int *test_cnt, cudaStream_t st);
cudaError_t launch_scan(const unsigned int *cnt, int64_t N, int64_t *off, cudaStream_t st);
cudaError_t launch_scatter(int64_t n, const double *x, const double *y, const uint8_t *role,
                           Axis ax, Axis ay, const int64_t *train_off, const int64_t *val_off,
                           const int64_t *test_off, unsigned int *train_cur, unsigned int *val_cur,
                           unsigned int *test_cur, int32_t *train_idx, int32_t *val_idx,
                           int32_t *test_idx, cudaStream_t st);
// Sort every segment of idx (ascending) whose length is <= max_len_small with one CTA
// per segment in shared memory; returns the padded power-of-two length used.
cudaError_t launch_segsort_small(int32_t *idx, const int64_t *off, int64_t N, int64_t max_len,
                                 cudaStream_t st);
// Sort one long segment [begin, begin+len) of distinct values in [0, n) via a bitmap.
cudaError_t sort_long_segment(int32_t *idx, int64_t begin, int64_t len, int64_t n,
                              uint32_t *bitmap, cudaStream_t st);
constexpr int64_t kSmallSortMax = 32768;
cudaError_t launch_gather(int64_t cnt, const int32_t *idx, const double *x, const double *y,
                          const double *v, double *ox, double *oy, double *ov, cudaStream_t st);

}  // namespace pgpcv
