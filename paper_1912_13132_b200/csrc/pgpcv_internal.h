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
    unsigned long long *counter;  // [1 + kMaxSms] zeroed before launch: claims (front | back << 32),
                                  // then per-SM CTA arrival counts
    int32_t sched;              // 0: every CTA claims from the front (LPT order); 1: the second
                                // CTA of each SM claims from the back (smallest k first)
    double *work;               // n_slots * slot_stride doubles: one factor per resident CTA
    size_t slot_stride;
    int32_t out_C;              // output row stride: entry (s, c) at s*out_C + (out_C > 1 ? c : 0)
    int32_t flags;              // kCvPredict | kCvNll
    int32_t border_pred;        // targets bordered below y (prediction without back-substitution):
                                // 0 never, 1 where 20 m <= k, 2 always
    double *subset_loss;        // [N*out_C] SSPE of the targets (kCvPredict)
    double *logdet;             // [N*out_C] sum_i log L_ii (kCvNll), for -2 log L (Eq.2)
    double *zz;                 // [N*out_C] ||L^{-1} y_T||^2 (kCvNll)
    double *yhat;               // [sum of targets] kriging predictions, or nullptr
    uint8_t *fail;              // [N*out_C] 1 = not positive definite
    // kCvGls (row f4): p covariate rows bordered below y; per-subset core-row sums
    int32_t p;                  // number of covariates (0 unless kCvGls)
    const double *tX;           // [sum_k * p] staged covariates of the training members
    const double *rects;        // [N*4] subset rectangles (the cores)
    double xmax, ymax;          // domain top edges (closed, R3)
    double *gls_out;            // [N * (p+1) * p]: A (p x p row-major) then b (p)
    unsigned long long *prof;   // [grid * 15] phase cycles (diagnostic build only) or nullptr
    unsigned long long *tl;     // [grid * 32768] GEMM/non-GEMM timeline (diagnostic) or nullptr
    // Per-range covariance reuse (small kernel only; DESIGN.md section 6 "K4s"): Sigma_theta
    // of each subset, generated once per call and range by sigma_kernel and read by every
    // (range, lambda) item of that subset instead of regenerating the exp/sqrt.  nullptr:
    // every item generates its own entries.
    const double *sig;          // [n_ranges * sig_stride] packed factor layout, ld = sigma_ld(k, nbt)
    const int64_t *sig_off;     // [N] offset (doubles) of subset s inside one range's block, -1: none
    size_t sig_stride;          // doubles per range block
    const int32_t *sig_range;   // [C] range index of config c
};

// Rows of the per-range covariance block of a subset: the k training rows, the y row
// (never read from it) and the nbt bordered target rows.
__host__ __device__ inline int64_t sigma_ld(int64_t k, int64_t nbt) { return ((k + nbt + 1 + 15) / 16) * 16; }
// Targets bordered below y by the small kernel (bordered prediction, border_pred 1: where
// 20 m <= k; 2: always), identical on the host and in both kernels.
__host__ __device__ inline int64_t border_rows(int32_t flags, int32_t border_pred, int64_t k, int64_t m) {
    return ((flags & 1) && (border_pred == 2 || (border_pred == 1 && 20 * m <= k))) ? m : 0;
}
cudaError_t launch_sigma(const int32_t *subs, int32_t n_subs, const double *ranges, int32_t n_ranges,
                         const int64_t *train_off, const int64_t *val_off, const double *tx, const double *ty,
                         const double *vx, const double *vy, int32_t flags, int32_t border_pred, double *sig,
                         const int64_t *sig_off, size_t sig_stride, cudaStream_t st);
// doubles of the packed per-range covariance block of a subset (column groups of 16 up to k)
int64_t sigma_doubles(int64_t k, int64_t nbt);
constexpr int32_t kCvPredict = 1;  // back-substitution, prediction, SSPE (Eq.3, Eq.4)
constexpr int32_t kCvNll = 2;      // -2 log-likelihood from the same factor (Eq.2)
constexpr int32_t kCvGls = 4;      // GLS normal-equation sums from the same factor (Eq. GLS)
constexpr int32_t kMaxCovariates = 8;
constexpr int kMaxSms = 256;
#define PGPCV_MAX_K_INTERNAL 65536  // must equal PGPCV_MAX_K in include/pgpcv.h

// Kernel geometry (see cv_kernel.cu for the derivation): two variants of the same kernel.
constexpr int kMT = 128;        // large: rows per row tile (8 warps)
constexpr int kNB = 64;         // large: block-column width of the left-looking Cholesky
constexpr int kMTSmall = 64;    // small: 4 warps
constexpr int kNBSmall = 32;
constexpr int kCvLarge = 0, kCvSmall = 1, kCvSmallSig = 2, kCvLargeWS = 3;  // kernel variants
constexpr int kCvVariants = 4;
int cv_kernel_slots_per_cta(int variant);  // factor slots (independent item streams) per CTA
size_t cv_kernel_smem_bytes(int variant);
int cv_kernel_max_k();
size_t cv_kernel_slot_doubles(int variant, int64_t kmax, int extra_rows = 0);  // factor + back-substitution scratch
// leading dimension (doubles) of a k-point factor: column-major (k+1) x k, +1 bordered row
__host__ __device__ inline int64_t factor_ld(int64_t k) { return ((k + 1 + 15) / 16) * 16; }

cudaError_t launch_cv_kernel(int variant, const CvArgs &a, int grid, cudaStream_t st);

// GLS (row f4): out[w] = sum_s part[s*W + w] in ascending s (W = (p+1) p), then
// beta = A^{-1} b by Gaussian elimination with partial pivoting; *status = 0 ok, 1 singular.
cudaError_t launch_gls_solve(const double *part, const uint8_t *fail, int64_t N, int32_t p, double *sums,
                             double *beta, int32_t *status, cudaStream_t st);
cudaError_t launch_gather_rows(int64_t cnt, const int32_t *idx, const double *X, int32_t p, double *out,
                               cudaStream_t st);
cudaError_t cv_kernel_occupancy(int variant, int *blocks_per_sm);
// zeta dedup: entry (s, c) <- unique-config entry (s, umap[c]) (stride U) where own[s], else
// 0; with nll: -2 log L_s = k log 2pi + k log sigma2_c + 2 logdet + zz / sigma2_c (Eq.2).
cudaError_t launch_expand(int64_t N, int32_t C, int32_t U, const int32_t *umap, const uint8_t *own,
                          const int64_t *train_off, const double *sigma2, const double *u_loss,
                          const uint8_t *u_fail, const double *u_logdet, const double *u_zz, double *loss,
                          uint8_t *fail, double *nll, cudaStream_t st);
// diagnostic: the CV kernel's elementary functions on device arrays (pgpcv_device_math)
cudaError_t launch_device_math(int32_t fn, int64_t n, const double *x, double *y, cudaStream_t st);
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

// Bisection tree (row f2): internal node id (1 = D, children 2i / 2i+1) splits along x at
// even depth and along y at odd depth at split[id]; rect[] holds the rectangles of the
// 2^depth nodes at `depth` (the leaves), as (x0, x1, y0, y1), closed at the domain top.
struct Tree {
    const double *split;  // [2^depth] (entry 0 unused)
    const double *rect;   // [2^depth * 4]
    int32_t depth;
    double xmax, ymax;
    double delta;
};

// Membership geometry of a partition: equal tiles (R1) or the leaves of a bisection tree.
struct Geom {
    int32_t kind;  // 0 grid, 1 tree
    Axis ax, ay;
    Tree tree;
};

#ifdef __CUDACC__
// R2/R3 dilated interval of [lo, hi): lo - delta <= u < hi + delta, hi = +inf at the top.
__device__ __forceinline__ bool in_dilated_iv(double u, double lo, double hi, double top, double delta) {
    const double l = __dsub_rn(lo, delta);
    const double h = hi == top ? __longlong_as_double(0x7ff0000000000000ll) : __dadd_rn(hi, delta);
    return l <= u && u < h;
}
// half-open core interval, closed at the domain top (R3)
__device__ __forceinline__ bool in_core_iv(double u, double lo, double hi, double top) {
    return lo <= u && (u < hi || (hi == top && u == top));
}
// f(leaf, in_dilated, in_core) for every leaf whose dilated rectangle contains (x, y).
// Descent prunes with u < c + delta (left) and u >= c - delta (right), both implied by the
// exact leaf test, so no member is lost; the leaf test itself decides.
template <class F>
__device__ __forceinline__ void tree_visit(const Tree &t, double x, double y, F f) {
    int stack[48];
    int sp = 0;
    stack[sp++] = 1;
    while (sp) {
        const int id = stack[--sp];
        const int dep = 31 - __clz(id);
        if (dep == t.depth) {
            const int s = id - (1 << t.depth);
            const double *r = t.rect + 4 * s;
            const bool dil = in_dilated_iv(x, r[0], r[1], t.xmax, t.delta) &&
                             in_dilated_iv(y, r[2], r[3], t.ymax, t.delta);
            if (dil) f(s, true, in_core_iv(x, r[0], r[1], t.xmax) && in_core_iv(y, r[2], r[3], t.ymax));
            continue;
        }
        const double c = t.split[id];
        const double u = (dep & 1) ? y : x;
        if (u >= __dsub_rn(c, t.delta)) stack[sp++] = 2 * id + 1;
        if (u < __dadd_rn(c, t.delta)) stack[sp++] = 2 * id;
    }
}
#endif

cudaError_t launch_validate(int64_t n, const double *x, const double *y, const double *v,
                            const uint8_t *role, double xmin, double xmax, double ymin,
                            double ymax, unsigned long long *stats, cudaStream_t st);
cudaError_t launch_count(int64_t n, const double *x, const double *y, const uint8_t *role,
                         const Geom &g, unsigned int *train_cnt, unsigned int *val_cnt,
                         unsigned int *test_cnt, cudaStream_t st);
cudaError_t launch_scan(const unsigned int *cnt, int64_t N, int64_t *off, cudaStream_t st);
cudaError_t launch_scatter(int64_t n, const double *x, const double *y, const uint8_t *role,
                           const Geom &g, const int64_t *train_off, const int64_t *val_off,
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

// ----------------------------------------------------------------------------------------
// Recursive shell-balanced bisection (row f2; bisect.cu).
// ----------------------------------------------------------------------------------------
// Computes split[1 .. 2^depth - 1] and the leaf rectangles rect[2^depth * 4] (device
// arrays, caller-allocated) for points with role <= 1, level by level; scratch comes from
// `pool` (stream-ordered; the ctx keeps it across calls).  Synchronises `st` once per level.
cudaError_t bisect_tree(int64_t n, const double *x, const double *y, const uint8_t *role, double xmin,
                        double xmax, double ymin, double ymax, int depth, double delta, double *split,
                        double *rect, cudaMemPool_t pool, cudaStream_t st);
// Shell cap (R22) on CSR training lists (ascending index) of N subsets with rectangles
// rect (device arrays): writes the capped lists (ascending index) to train_idx_out /
// train_off_out (device, capacity sum_k / N+1) and the number of dropped members to
// *n_dropped (host).  Synchronises `st`.
cudaError_t cap_shells(int64_t N, const int64_t *train_off, const int32_t *train_idx, const double *x,
                       const double *y, const double *rect, double xmax, double ymax, int64_t cap, uint64_t seed,
                       int32_t *train_idx_out, int64_t *train_off_out, int64_t *n_dropped, cudaMemPool_t pool,
                       cudaStream_t st);

}  // namespace pgpcv
