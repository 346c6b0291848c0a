// bisect.cu -- row f2 of the scope table: the paper's own division of the data into
// subsets (§2.4) and the shell cap of §4.3.2.
//
// Recursive shell-balanced bisection (readings R19-R21 in DESIGN.md): node 1 = D; a node
// at depth d is split along x (d even) or y (d odd) by the line c that minimises
// |count_left - count_right|, where a child's count is the number of training and
// validation points in its L-inf dilation by delta (the child "together with its shell",
// P:247); candidates are c = 0.5 (u_j + u_{j+1}) for consecutive distinct split
// coordinates u_j < u_{j+1} of counted points in the node's core; ties go to the smaller
// c; a node without a candidate splits at its midpoint.
//
// One level at a time, all nodes of the level in parallel:
//   B1 count   -- every counted point visits the nodes whose dilated rectangle holds it
//                 (tree descent, exact R2/R3 test at the node) and counts band / core
//   B2 scan    -- CSR offsets (the partition's single-CTA scan)
//   B3 scatter -- split coordinates into per-node band and core segments
//   B4 sort    -- CUB segmented sort of both (a library sort: this runs once per dataset,
//                 outside the per-configuration hot path)
//   B5 score   -- one thread per candidate: two binary searches in the sorted band give
//                 count_left = #{u < c + delta} and count_right = #{u >= c - delta};
//                 (score, j) packed in 64 bits and atomicMin'ed per node
//   B6 split   -- per node: the winning c (or the midpoint) -> split[id], child rects
// Every comparison is an exact FP64 comparison and c, c +- delta are single correctly
// rounded operations, so the tree is bit-identical to the oracle's.
//
// Shell cap (R22): in a subset whose shell (training members outside the core rectangle)
// exceeds `cap`, keep the `cap` shell members with the smallest SplitMix64 keys
// key(s, p) = splitmix64(seed, s 2^32 + p + 1) (ties: smaller p); core members are kept.
#include <cub/device/device_segmented_sort.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "pgpcv_internal.h"

namespace pgpcv {
namespace {

inline int grid_for(int64_t n) {
    int64_t b = (n + 255) / 256;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32));
}

// B1 / B3: band (dilated rectangle) and core memberships of counted points at this level.
__global__ void band_kernel(int64_t n, const double *x, const double *y, const uint8_t *role, Tree t, int axis,
                            unsigned int *band_cnt, unsigned int *core_cnt, const int64_t *band_off,
                            const int64_t *core_off, double *band, double *core) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        if (role[p] > 1) continue;  // test points never count (R20)
        const double px = x[p], py = y[p];
        const double u = axis ? py : px;
        tree_visit(t, px, py, [&](int s, bool, bool incore) {
            if (!band) {
                atomicAdd(band_cnt + s, 1u);
                if (incore) atomicAdd(core_cnt + s, 1u);
            } else {
                band[band_off[s] + atomicAdd(band_cnt + s, 1u)] = u;
                if (incore) core[core_off[s] + atomicAdd(core_cnt + s, 1u)] = u;
            }
        });
    }
}

__device__ __forceinline__ int64_t count_below(const double *a, int64_t len, double v) {
    int64_t lo = 0, hi = len;
    while (lo < hi) {
        const int64_t mid = lo + ((hi - lo) >> 1);
        if (a[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// B5: one thread per candidate position j of the concatenated sorted core segments.
__global__ void score_kernel(const double *band, const int64_t *band_off, const double *core, const int64_t *core_off,
                             int64_t nodes, int64_t total_core, double delta, unsigned long long *best) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < total_core;
         j += (int64_t)gridDim.x * blockDim.x) {
        // node of j: the last s with core_off[s] <= j
        int64_t lo = 0, hi = nodes - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (core_off[mid] <= j) lo = mid;
            else hi = mid - 1;
        }
        const int64_t s = lo;
        if (j + 1 >= core_off[s + 1]) continue;  // last core value of the node
        const double u0 = core[j], u1 = core[j + 1];
        if (!(u0 < u1)) continue;  // not distinct
        const double c = __dmul_rn(0.5, __dadd_rn(u0, u1));
        const double *b = band + band_off[s];
        const int64_t nb = band_off[s + 1] - band_off[s];
        const int64_t left = count_below(b, nb, __dadd_rn(c, delta));
        const int64_t right = nb - count_below(b, nb, __dsub_rn(c, delta));
        const unsigned long long score = (unsigned long long)(left > right ? left - right : right - left);
        const unsigned long long jl = (unsigned long long)(j - core_off[s]);
        atomicMin(best + s, (score << 32) | jl);  // ties: smallest j = smallest c
    }
}

// B6: split value of every node of the level and the rectangles of the next level.
__global__ void split_kernel(const double *core, const int64_t *core_off, const unsigned long long *best,
                             const double *rect, int64_t nodes, int axis, int64_t first_id, double *split,
                             double *next_rect) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= nodes) return;
    const double *r = rect + 4 * s;
    double c;
    if (best[s] == ~0ull) {
        c = __dmul_rn(0.5, __dadd_rn(r[2 * axis], r[2 * axis + 1]));  // R21: no candidate
    } else {
        const int64_t j = core_off[s] + (int64_t)(best[s] & 0xffffffffull);
        c = __dmul_rn(0.5, __dadd_rn(core[j], core[j + 1]));
    }
    split[first_id + s] = c;
    double *lc = next_rect + 4 * (2 * s), *rc = next_rect + 4 * (2 * s + 1);
    for (int i = 0; i < 4; ++i) lc[i] = rc[i] = r[i];
    lc[2 * axis + 1] = c;
    rc[2 * axis] = c;
}

// ---------------------------------------------------------------- shell cap
__device__ __forceinline__ uint64_t splitmix64(uint64_t seed, uint64_t i) {
    uint64_t z = seed + i * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// One CTA per subset: flag shell members (outside the core rectangle), count them.
__global__ void shell_flag_kernel(const int64_t *off, const int32_t *idx, const double *x, const double *y,
                                  const double *rect, double xmax, double ymax, uint8_t *is_shell,
                                  unsigned int *shell_cnt) {
    const int64_t s = blockIdx.x;
    const double *r = rect + 4 * s;
    unsigned int cnt = 0;
    for (int64_t i = off[s] + threadIdx.x; i < off[s + 1]; i += blockDim.x) {
        const int32_t p = idx[i];
        const bool core = in_core_iv(x[p], r[0], r[1], xmax) && in_core_iv(y[p], r[2], r[3], ymax);
        is_shell[i] = !core;
        cnt += !core;
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(shell_cnt + s, cnt);
}

// Gather the shell members of the capped subsets, in list order, with their keys.  One
// CTA per capped subset; a block-wide running count keeps the order stable.
__global__ void shell_gather_kernel(const int64_t *off, const int32_t *idx, const uint8_t *is_shell,
                                    const int32_t *capped, const int64_t *seg_off, uint64_t seed, uint64_t *keys,
                                    int64_t *pos) {
    __shared__ unsigned int warp_cnt[32];
    __shared__ int64_t base;
    const int64_t s = capped[blockIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) base = seg_off[blockIdx.x];
    __syncthreads();
    for (int64_t i0 = off[s]; i0 < off[s + 1]; i0 += blockDim.x) {
        const int64_t i = i0 + threadIdx.x;
        const bool f = i < off[s + 1] && is_shell[i];
        const unsigned int m = __ballot_sync(0xffffffffu, f);
        if (lane == 0) warp_cnt[warp] = __popc(m);
        __syncthreads();
        int64_t before = base;
        for (int w = 0; w < warp; ++w) before += warp_cnt[w];
        if (f) {
            const int64_t o = before + __popc(m & ((1u << lane) - 1u));
            keys[o] = splitmix64(seed, ((uint64_t)s << 32) + (uint64_t)idx[i] + 1ull);
            pos[o] = i;
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int w = 0; w < nw; ++w) base += warp_cnt[w];
        __syncthreads();
    }
}

// Members of rank >= cap in their (key, position)-sorted shell segment are dropped.
__global__ void shell_drop_kernel(const int64_t *seg_off, int64_t nseg, const int64_t *pos_sorted, int64_t cap,
                                  uint8_t *keep) {
    const int64_t g = blockIdx.x;
    if (g >= nseg) return;
    for (int64_t r = seg_off[g] + cap + threadIdx.x; r < seg_off[g + 1]; r += blockDim.x) keep[pos_sorted[r]] = 0;
}

__global__ void kept_count_kernel(const int64_t *off, const uint8_t *keep, int64_t N, int64_t *cnt) {
    const int64_t s = blockIdx.x;
    if (s >= N) return;
    unsigned int c = 0;
    for (int64_t i = off[s] + threadIdx.x; i < off[s + 1]; i += blockDim.x) c += keep[i];
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    __shared__ unsigned int part[32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
        cnt[s] = t;
    }
}

struct Scratch {  // stream-ordered temporaries of one call, from the ctx's own pool
    cudaStream_t st;
    cudaMemPool_t pool;
    std::vector<void *> ptrs;
    Scratch(cudaStream_t s, cudaMemPool_t p) : st(s), pool(p) {}
    ~Scratch() {
        for (void *p : ptrs) cudaFreeAsync(p, st);
    }
    template <class T>
    cudaError_t get(T **out, size_t count) {
        void *p = nullptr;
        cudaError_t e = pool ? cudaMallocFromPoolAsync(&p, std::max<size_t>(count, 1) * sizeof(T), pool, st)
                             : cudaMallocAsync(&p, std::max<size_t>(count, 1) * sizeof(T), st);
        if (e != cudaSuccess) return e;
        ptrs.push_back(p);
        *out = (T *)p;
        return cudaSuccess;
    }
};

#define RET(x)                                \
    do {                                      \
        cudaError_t e_ = (x);                 \
        if (e_ != cudaSuccess) return e_;     \
    } while (0)

// exclusive scan of `cnt` (unsigned) into off[0..N] on the host (N <= 2^20 nodes)
cudaError_t scan_to_host_and_device(const unsigned int *d_cnt, int64_t N, int64_t *d_off, std::vector<int64_t> &h_off,
                                    cudaStream_t st) {
    std::vector<unsigned int> h(N);
    RET(cudaMemcpyAsync(h.data(), d_cnt, sizeof(unsigned) * N, cudaMemcpyDeviceToHost, st));
    RET(cudaStreamSynchronize(st));
    h_off.assign(N + 1, 0);
    for (int64_t i = 0; i < N; ++i) h_off[i + 1] = h_off[i] + h[i];
    return cudaMemcpyAsync(d_off, h_off.data(), sizeof(int64_t) * (N + 1), cudaMemcpyHostToDevice, st);
}

}  // namespace

cudaError_t bisect_tree(int64_t n, const double *x, const double *y, const uint8_t *role, double xmin, double xmax,
                        double ymin, double ymax, int depth, double delta, double *split, double *rect,
                        cudaMemPool_t pool, cudaStream_t st) {
    Scratch S(st, pool);
    const int64_t N = (int64_t)1 << depth;
    double *lvl_rect, *next_rect;
    RET(S.get(&lvl_rect, 4 * N));
    RET(S.get(&next_rect, 4 * N));
    const double root[4] = {xmin, xmax, ymin, ymax};
    RET(cudaMemcpyAsync(lvl_rect, root, sizeof root, cudaMemcpyHostToDevice, st));
    RET(cudaMemsetAsync(split, 0, sizeof(double) * N, st));
    unsigned int *band_cnt, *core_cnt;
    int64_t *band_off, *core_off;
    unsigned long long *best;
    RET(S.get(&band_cnt, N));
    RET(S.get(&core_cnt, N));
    RET(S.get(&band_off, N + 1));
    RET(S.get(&core_off, N + 1));
    RET(S.get(&best, N));
    for (int d = 0; d < depth; ++d) {
        const int64_t nodes = (int64_t)1 << d;
        const int axis = d & 1;
        Tree t{split, lvl_rect, d, xmax, ymax, delta};
        RET(cudaMemsetAsync(band_cnt, 0, sizeof(unsigned) * nodes, st));
        RET(cudaMemsetAsync(core_cnt, 0, sizeof(unsigned) * nodes, st));
        band_kernel<<<grid_for(n), 256, 0, st>>>(n, x, y, role, t, axis, band_cnt, core_cnt, nullptr, nullptr,
                                                 nullptr, nullptr);
        RET(cudaGetLastError());
        std::vector<int64_t> hb, hc;
        RET(scan_to_host_and_device(band_cnt, nodes, band_off, hb, st));
        RET(scan_to_host_and_device(core_cnt, nodes, core_off, hc, st));
        const int64_t nb = hb[nodes], nc = hc[nodes];
        double *band, *core, *band_s, *core_s;
        RET(S.get(&band, nb));
        RET(S.get(&core, nc));
        RET(S.get(&band_s, nb));
        RET(S.get(&core_s, nc));
        RET(cudaMemsetAsync(band_cnt, 0, sizeof(unsigned) * nodes, st));
        RET(cudaMemsetAsync(core_cnt, 0, sizeof(unsigned) * nodes, st));
        band_kernel<<<grid_for(n), 256, 0, st>>>(n, x, y, role, t, axis, band_cnt, core_cnt, band_off, core_off,
                                                 band, core);
        RET(cudaGetLastError());
        // B4: CUB segmented sorts (library primitive)
        size_t tb = 0, tc = 0;
        if (nb > 0)
            RET(cub::DeviceSegmentedSort::SortKeys(nullptr, tb, band, band_s, (int)nb, (int)nodes, band_off,
                                                   band_off + 1, st));
        if (nc > 0)
            RET(cub::DeviceSegmentedSort::SortKeys(nullptr, tc, core, core_s, (int)nc, (int)nodes, core_off,
                                                   core_off + 1, st));
        void *tmp;
        RET(S.get((uint8_t **)&tmp, std::max(tb, tc)));
        if (nb > 0)
            RET(cub::DeviceSegmentedSort::SortKeys(tmp, tb, band, band_s, (int)nb, (int)nodes, band_off,
                                                   band_off + 1, st));
        if (nc > 0)
            RET(cub::DeviceSegmentedSort::SortKeys(tmp, tc, core, core_s, (int)nc, (int)nodes, core_off,
                                                   core_off + 1, st));
        RET(cudaMemsetAsync(best, 0xff, sizeof(unsigned long long) * nodes, st));
        if (nc > 0) {
            score_kernel<<<grid_for(nc), 256, 0, st>>>(band_s, band_off, core_s, core_off, nodes, nc, delta, best);
            RET(cudaGetLastError());
        }
        split_kernel<<<(unsigned)((nodes + 127) / 128), 128, 0, st>>>(core_s, core_off, best, lvl_rect, nodes, axis,
                                                                      nodes, split, next_rect);
        RET(cudaGetLastError());
        std::swap(lvl_rect, next_rect);
        RET(cudaStreamSynchronize(st));
    }
    return cudaMemcpyAsync(rect, lvl_rect, sizeof(double) * 4 * N, cudaMemcpyDeviceToDevice, st);
}

cudaError_t cap_shells(int64_t N, const int64_t *train_off, const int32_t *train_idx, const double *x,
                       const double *y, const double *rect, double xmax, double ymax, int64_t cap, uint64_t seed,
                       int32_t *train_idx_out, int64_t *train_off_out, int64_t *n_dropped, cudaMemPool_t pool,
                       cudaStream_t st) {
    Scratch S(st, pool);
    std::vector<int64_t> hoff(N + 1);
    RET(cudaMemcpyAsync(hoff.data(), train_off, sizeof(int64_t) * (N + 1), cudaMemcpyDeviceToHost, st));
    RET(cudaStreamSynchronize(st));
    const int64_t total = hoff[N];
    uint8_t *is_shell, *keep;
    unsigned int *shell_cnt;
    RET(S.get(&is_shell, total));
    RET(S.get(&keep, total));
    RET(S.get(&shell_cnt, N));
    RET(cudaMemsetAsync(shell_cnt, 0, sizeof(unsigned) * N, st));
    RET(cudaMemsetAsync(keep, 1, total, st));
    if (N > 0) shell_flag_kernel<<<(unsigned)N, 256, 0, st>>>(train_off, train_idx, x, y, rect, xmax, ymax,
                                                               is_shell, shell_cnt);
    RET(cudaGetLastError());
    std::vector<unsigned int> hshell(N);
    RET(cudaMemcpyAsync(hshell.data(), shell_cnt, sizeof(unsigned) * N, cudaMemcpyDeviceToHost, st));
    RET(cudaStreamSynchronize(st));
    std::vector<int32_t> capped;
    std::vector<int64_t> seg{0};
    for (int64_t s = 0; s < N; ++s)
        if ((int64_t)hshell[s] > cap) {
            capped.push_back((int32_t)s);
            seg.push_back(seg.back() + hshell[s]);
        }
    int64_t dropped = 0;
    for (int32_t s : capped) dropped += (int64_t)hshell[s] - cap;
    *n_dropped = dropped;
    if (!capped.empty()) {
        const int64_t nseg = (int64_t)capped.size(), m = seg.back();
        int32_t *d_capped;
        int64_t *d_seg, *pos, *pos_s;
        uint64_t *keys, *keys_s;
        RET(S.get(&d_capped, nseg));
        RET(S.get(&d_seg, nseg + 1));
        RET(S.get(&keys, m));
        RET(S.get(&keys_s, m));
        RET(S.get(&pos, m));
        RET(S.get(&pos_s, m));
        RET(cudaMemcpyAsync(d_capped, capped.data(), sizeof(int32_t) * nseg, cudaMemcpyHostToDevice, st));
        RET(cudaMemcpyAsync(d_seg, seg.data(), sizeof(int64_t) * (nseg + 1), cudaMemcpyHostToDevice, st));
        shell_gather_kernel<<<(unsigned)nseg, 256, 0, st>>>(train_off, train_idx, is_shell, d_capped, d_seg, seed,
                                                            keys, pos);
        RET(cudaGetLastError());
        // stable: equal keys keep list order, i.e. ascending point index (R22 tie rule)
        size_t tb = 0;
        RET(cub::DeviceSegmentedSort::StableSortPairs(nullptr, tb, keys, keys_s, pos, pos_s, (int)m, (int)nseg,
                                                      d_seg, d_seg + 1, st));
        uint8_t *tmp;
        RET(S.get(&tmp, tb));
        RET(cub::DeviceSegmentedSort::StableSortPairs(tmp, tb, keys, keys_s, pos, pos_s, (int)m, (int)nseg, d_seg,
                                                      d_seg + 1, st));
        shell_drop_kernel<<<(unsigned)nseg, 256, 0, st>>>(d_seg, nseg, pos_s, cap, keep);
        RET(cudaGetLastError());
    }
    // new offsets and the stable compaction (ascending index order is preserved)
    int64_t *cnt;
    RET(S.get(&cnt, N));
    if (N > 0) kept_count_kernel<<<(unsigned)N, 256, 0, st>>>(train_off, keep, N, cnt);
    RET(cudaGetLastError());
    std::vector<int64_t> hc(N), noff(N + 1, 0);
    RET(cudaMemcpyAsync(hc.data(), cnt, sizeof(int64_t) * N, cudaMemcpyDeviceToHost, st));
    RET(cudaStreamSynchronize(st));
    for (int64_t s = 0; s < N; ++s) noff[s + 1] = noff[s] + hc[s];
    RET(cudaMemcpyAsync(train_off_out, noff.data(), sizeof(int64_t) * (N + 1), cudaMemcpyHostToDevice, st));
    int64_t *nsel;
    RET(S.get(&nsel, 1));
    size_t tb = 0;
    RET(cub::DeviceSelect::Flagged(nullptr, tb, train_idx, keep, train_idx_out, nsel, total, st));
    uint8_t *tmp;
    RET(S.get(&tmp, tb));
    RET(cub::DeviceSelect::Flagged(tmp, tb, train_idx, keep, train_idx_out, nsel, total, st));
    return cudaStreamSynchronize(st);
}

}  // namespace pgpcv
