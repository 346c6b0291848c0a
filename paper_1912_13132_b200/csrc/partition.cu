// partition.cu -- Alg.1 lines 2-3: divide the data into the
// training subsets y~^i_T (core tile plus shell of width delta) and the
// validation subsets y^i_V (core tile only, Eq.7), once per dataset.
//
// Membership is decided by FP64 comparisons only, against edge/bound arrays the host
// computes with the DESIGN.md R4 formulas, so the result is bit-exact and independent of
// device arithmetic.  Because lo_i = e_i - delta and hi_i = e_{i+1} + delta are
// non-decreasing in i, {i : lo_i <= x < hi_i} is an interval, found by two binary
// searches; the core tile is the largest i with e_i <= x (clamped to K-1 at the closed
// top edge).  Counting sort: count (K1) -> exclusive scan (K2) -> scatter (K3) ->
// per-segment ascending sort (K3b) -> staging gather (K4).
#include <cmath>
#include <cstdint>

#include "pgpcv_internal.h"

namespace pgpcv {
namespace {

// largest i in [0, K-1] with e[i] <= x
__device__ __forceinline__ int core_index(double x, const double *e, int K) {
    int lo = 0, hi = K - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (e[mid] <= x) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// [first, last] = {i : lo[i] <= x < hi[i]} (empty if first > last)
__device__ __forceinline__ int2 dilated_range(double x, const Axis &a) {
    int l = 0, h = a.K;  // first i with x < hi[i]  (hi non-decreasing, hi[K-1] = +inf)
    while (l < h) {
        const int mid = (l + h) >> 1;
        if (x < a.hi[mid]) h = mid;
        else l = mid + 1;
    }
    const int first = l;
    l = -1;
    h = a.K - 1;  // last i with lo[i] <= x  (lo non-decreasing)
    while (l < h) {
        const int mid = (l + h + 1) >> 1;
        if (a.lo[mid] <= x) l = mid;
        else h = mid - 1;
    }
    return make_int2(first, l);
}

__global__ void validate_kernel(int64_t n, const double *x, const double *y, const double *v,
                                const uint8_t *role, double xmin, double xmax, double ymin,
                                double ymax, unsigned long long *stats) {
    unsigned long long f = 0, nt = 0, nv = 0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const double px = x[p], py = y[p], pv = v[p];
        if (!isfinite(px) || !isfinite(py) || !isfinite(pv)) f |= 1u;
        else if (px < xmin || px > xmax || py < ymin || py > ymax) f |= 2u;
        const uint8_t r = role[p];
        if (r > 2) f |= 4u;
        nt += r == 0;
        nv += r == 1;
    }
    if (f) atomicOr(stats, f);
    if (nt) atomicAdd(stats + 1, nt);
    if (nv) atomicAdd(stats + 2, nv);
}

// Visit the memberships of point (px, py) with role r under geometry g:
//   r == 0: every subset whose dilated tile/rectangle holds the point (training, y~^s_T)
//   r == 1 / 2: the core tile/rectangle (validation y^s_V / test targets)
template <class F>
__device__ __forceinline__ void for_each_member(const Geom &g, double px, double py, uint8_t r, F f) {
    if (g.kind == 0) {
        if (r == 1 || r == 2) {
            const int ix = core_index(px, g.ax.e, g.ax.K), iy = core_index(py, g.ay.e, g.ay.K);
            f((int64_t)iy * g.ax.K + ix);
        } else if (r == 0) {
            const int2 rx = dilated_range(px, g.ax), ry = dilated_range(py, g.ay);
            for (int iy = ry.x; iy <= ry.y; ++iy)
                for (int ix = rx.x; ix <= rx.y; ++ix) f((int64_t)iy * g.ax.K + ix);
        }
    } else if (r <= 2) {
        tree_visit(g.tree, px, py, [&](int s, bool, bool core) {
            if (r == 0 || core) f((int64_t)s);
        });
    }
}

__global__ void count_kernel(int64_t n, const double *x, const double *y, const uint8_t *role, Geom g,
                             unsigned int *train_cnt, unsigned int *val_cnt, unsigned int *test_cnt) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t r = role[p];
        unsigned int *cnt = r == 0 ? train_cnt : r == 1 ? val_cnt : test_cnt;
        for_each_member(g, x[p], y[p], r, [&](int64_t s) { atomicAdd(cnt + s, 1u); });
    }
}

__global__ void scatter_kernel(int64_t n, const double *x, const double *y, const uint8_t *role, Geom g,
                               const int64_t *train_off, const int64_t *val_off, const int64_t *test_off,
                               unsigned int *train_cur, unsigned int *val_cur, unsigned int *test_cur,
                               int32_t *train_idx, int32_t *val_idx, int32_t *test_idx) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t r = role[p];
        const int64_t *off = r == 0 ? train_off : r == 1 ? val_off : test_off;
        unsigned int *cur = r == 0 ? train_cur : r == 1 ? val_cur : test_cur;
        int32_t *idx = r == 0 ? train_idx : r == 1 ? val_idx : test_idx;
        for_each_member(g, x[p], y[p], r, [&](int64_t s) { idx[off[s] + atomicAdd(cur + s, 1u)] = (int32_t)p; });
    }
}

// Exclusive scan of N counts into off[0..N] with one CTA (N <= a few 1e5).
__global__ void scan_kernel(const unsigned int *cnt, int64_t N, int64_t *off) {
    __shared__ int64_t part[1024];
    const int tid = threadIdx.x;
    const int64_t per = (N + blockDim.x - 1) / blockDim.x;
    const int64_t b = tid * per, e = min(N, b + per);
    int64_t sum = 0;
    for (int64_t i = b; i < e; ++i) sum += cnt[i];
    part[tid] = sum;
    __syncthreads();
    if (tid == 0) {
        int64_t run = 0;
        for (int i = 0; i < (int)blockDim.x; ++i) {
            const int64_t v = part[i];
            part[i] = run;
            run += v;
        }
        off[N] = run;
    }
    __syncthreads();
    int64_t run = part[tid];
    for (int64_t i = b; i < e; ++i) {
        off[i] = run;
        run += cnt[i];
    }
}

// One CTA per segment: bitonic sort of the segment in shared memory (padded with INT_MAX
// to the power-of-two length P).
__global__ void segsort_kernel(int32_t *idx, const int64_t *off, int P) {
    extern __shared__ int32_t keys[];
    const int64_t b = off[blockIdx.x], len = off[blockIdx.x + 1] - b;
    if (len <= 1 || len > P) return;
    for (int i = threadIdx.x; i < P; i += blockDim.x) keys[i] = i < len ? idx[b + i] : 0x7fffffff;
    __syncthreads();
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < P / 2; i += blockDim.x) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool up = (lo & size) == 0;
                const int32_t a = keys[lo], c = keys[hi];
                if ((a > c) == up) {
                    keys[lo] = c;
                    keys[hi] = a;
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < len; i += blockDim.x) idx[b + i] = keys[i];
}

__global__ void bitmap_set_kernel(const int32_t *idx, int64_t len, uint32_t *bm) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t p = idx[i];
        atomicOr(bm + (p >> 5), 1u << (p & 31));
    }
}

// One CTA: compact the set bits of bm (nwords words) into out[] in ascending order.
__global__ void bitmap_compact_kernel(const uint32_t *bm, int64_t nwords, int32_t *out) {
    __shared__ int64_t part[1024];
    const int tid = threadIdx.x;
    const int64_t per = (nwords + blockDim.x - 1) / blockDim.x;
    const int64_t b = tid * per, e = min(nwords, b + per);
    int64_t cnt = 0;
    for (int64_t w = b; w < e; ++w) cnt += __popc(bm[w]);
    part[tid] = cnt;
    __syncthreads();
    if (tid == 0) {
        int64_t run = 0;
        for (int i = 0; i < (int)blockDim.x; ++i) {
            const int64_t v = part[i];
            part[i] = run;
            run += v;
        }
    }
    __syncthreads();
    int64_t pos = part[tid];
    for (int64_t w = b; w < e; ++w) {
        uint32_t bits = bm[w];
        while (bits) {
            const int bit = __ffs(bits) - 1;
            out[pos++] = (int32_t)(w * 32 + bit);
            bits &= bits - 1;
        }
    }
}

__global__ void gather_kernel(int64_t cnt, const int32_t *idx, const double *x, const double *y,
                              const double *v, double *ox, double *oy, double *ov) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t p = idx[i];
        ox[i] = x[p];
        oy[i] = y[p];
        ov[i] = v[p];
    }
}

inline int grid_for(int64_t n) {
    int64_t b = (n + 255) / 256;
    if (b < 1) b = 1;
    if (b > 148 * 32) b = 148 * 32;
    return (int)b;
}

}  // namespace

cudaError_t launch_validate(int64_t n, const double *x, const double *y, const double *v,
                            const uint8_t *role, double xmin, double xmax, double ymin,
                            double ymax, unsigned long long *stats, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    validate_kernel<<<grid_for(n), 256, 0, st>>>(n, x, y, v, role, xmin, xmax, ymin, ymax, stats);
    return cudaGetLastError();
}

cudaError_t launch_count(int64_t n, const double *x, const double *y, const uint8_t *role,
                         const Geom &g, unsigned int *train_cnt, unsigned int *val_cnt,
                         unsigned int *test_cnt, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    count_kernel<<<grid_for(n), 256, 0, st>>>(n, x, y, role, g, train_cnt, val_cnt, test_cnt);
    return cudaGetLastError();
}

cudaError_t launch_scan(const unsigned int *cnt, int64_t N, int64_t *off, cudaStream_t st) {
    scan_kernel<<<1, 1024, 0, st>>>(cnt, N, off);
    return cudaGetLastError();
}

cudaError_t launch_scatter(int64_t n, const double *x, const double *y, const uint8_t *role,
                           const Geom &g, const int64_t *train_off, const int64_t *val_off,
                           const int64_t *test_off, unsigned int *train_cur, unsigned int *val_cur,
                           unsigned int *test_cur, int32_t *train_idx, int32_t *val_idx,
                           int32_t *test_idx, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    scatter_kernel<<<grid_for(n), 256, 0, st>>>(n, x, y, role, g, train_off, val_off, test_off,
                                                train_cur, val_cur, test_cur, train_idx, val_idx,
                                                test_idx);
    return cudaGetLastError();
}

cudaError_t launch_segsort_small(int32_t *idx, const int64_t *off, int64_t N, int64_t max_len,
                                 cudaStream_t st) {
    if (N == 0 || max_len <= 1) return cudaSuccess;
    int P = 2;
    while (P < max_len && P < kSmallSortMax) P <<= 1;
    const size_t smem = sizeof(int32_t) * (size_t)P;
    cudaError_t e = cudaFuncSetAttribute(segsort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    segsort_kernel<<<(unsigned)N, 1024, smem, st>>>(idx, off, P);
    return cudaGetLastError();
}

cudaError_t sort_long_segment(int32_t *idx, int64_t begin, int64_t len, int64_t n,
                              uint32_t *bitmap, cudaStream_t st) {
    const int64_t nwords = (n + 31) / 32;
    cudaError_t e = cudaMemsetAsync(bitmap, 0, sizeof(uint32_t) * nwords, st);
    if (e != cudaSuccess) return e;
    bitmap_set_kernel<<<grid_for(len), 256, 0, st>>>(idx + begin, len, bitmap);
    bitmap_compact_kernel<<<1, 1024, 0, st>>>(bitmap, nwords, idx + begin);
    return cudaGetLastError();
}

cudaError_t launch_gather(int64_t cnt, const int32_t *idx, const double *x, const double *y,
                          const double *v, double *ox, double *oy, double *ov, cudaStream_t st) {
    if (cnt == 0) return cudaSuccess;
    gather_kernel<<<grid_for(cnt), 256, 0, st>>>(cnt, idx, x, y, v, ox, oy, ov);
    return cudaGetLastError();
}

}  // namespace pgpcv
