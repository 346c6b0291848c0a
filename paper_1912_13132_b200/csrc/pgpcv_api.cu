// pgpcv_api.cu -- the C ABI of libpgpcv (include/pgpcv.h): argument checking, device
// memory and stream ownership, work scheduling (LPT), the NCCL combine step, timing.
// Every numerical step runs in the kernels of partition.cu and cv_kernel.cu.
#include <dlfcn.h>
#include <sched.h>
#include <time.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include <nccl.h>

#include "../../include/pgpcv.h"
#include <nvtx3/nvToolsExt.h>
#include "pgpcv_internal.h"

using namespace pgpcv;

namespace {

// NVTX range over a scope (an nsys / ncu timeline shows each API call and the phases of an
// evaluation by name; header-only NVTX v3, a no-op unless a tool is attached).
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

// ------------------------------------------------------------------ device buffers
template <typename T>
struct DevBuf {
    T *p = nullptr;
    size_t cap = 0;  // elements
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() { release(); }
    void swap(DevBuf &o) {
        std::swap(p, o.p);
        std::swap(cap, o.cap);
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    // grow-only; returns cudaSuccess or the allocation error
    cudaError_t ensure(size_t count) {
        if (count <= cap && p) return cudaSuccess;
        release();
        size_t bytes = sizeof(T) * std::max<size_t>(count, 1);
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess) {
            p = nullptr;
            cudaGetLastError();
            return e;
        }
        cap = std::max<size_t>(count, 1);
        return cudaSuccess;
    }
};

// ------------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
    bool ok = false;
    std::string why;
    std::string where;  // the bound library: path (dladdr) and version, or why none
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                              ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*commAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*commGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
    ncclResult_t (*getVersion)(int *) = nullptr;
    const char *(*getErrorString)(ncclResult_t) = nullptr;
};

// Any already-loaded object that exports ncclGetUniqueId (torch's libtorch_cuda links its
// bundled NCCL statically or as libnccl.so.2): reuse it so one process never holds two NCCLs.
void *nccl_already_loaded() {
    if (void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD)) return h;
    if (dlsym(RTLD_DEFAULT, "ncclGetUniqueId")) return RTLD_DEFAULT;
    return nullptr;
}

NcclApi &nccl() {
    static NcclApi api;
    static bool tried = false;
    if (tried) return api;
    tried = true;
    // PGPCV_NCCL_LIB, when set, is an explicit choice and is bound first, privately
    // (RTLD_LOCAL: it never interposes on an NCCL the process already holds); otherwise an
    // already-loaded NCCL is reused, else libnccl.so.2 is loaded.
    void *h = nullptr;
    if (const char *env = getenv("PGPCV_NCCL_LIB")) h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
    if (!h) h = nccl_already_loaded();
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        api.why = std::string("cannot dlopen libnccl.so.2: ") + dlerror();
        api.where = api.why;
        return api;
    }
    api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
    api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
    api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
    api.commAbort = (decltype(api.commAbort))dlsym(h, "ncclCommAbort");
    api.commGetAsyncError = (decltype(api.commGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
    api.getVersion = (decltype(api.getVersion))dlsym(h, "ncclGetVersion");
    api.getErrorString = (decltype(api.getErrorString))dlsym(h, "ncclGetErrorString");
    api.ok = api.getUniqueId && api.commInitRank && api.allReduce && api.commDestroy && api.commAbort &&
             api.commGetAsyncError && api.getVersion && api.getErrorString;
    if (!api.ok) {
        api.why = "libnccl.so.2 lacks a required symbol";
        api.where = api.why;
        return api;
    }
    Dl_info info{};
    const char *path = dladdr((void *)api.getUniqueId, &info) && info.dli_fname ? info.dli_fname : "?";
    int v = 0;
    api.getVersion(&v);
    char buf[1024];
    snprintf(buf, sizeof buf, "%s (NCCL %d.%d.%d)", path, v / 10000, (v / 100) % 100, v % 100);
    api.where = buf;
    if (getenv("PGPCV_VERBOSE")) fprintf(stderr, "libpgpcv: NCCL bound from %s\n", buf);
    return api;
}

double now_s() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

std::string g_create_error;

// status: -1 -> INT32_MAX so a MIN all-reduce yields the smallest failing subset, and back
__global__ void status_encode(int32_t *st, int32_t C, int32_t sentinel) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < C && st[c] == sentinel) st[c] = (sentinel == -1) ? 0x7fffffff : -1;
}
cudaError_t launch_status_encode(int32_t *st, int32_t C, int32_t sentinel, cudaStream_t stream) {
    status_encode<<<(C + 127) / 128, 128, 0, stream>>>(st, C, sentinel);
    return cudaGetLastError();
}

// R4: e_i = a + i*w (separate multiply and add), e_K = b; bounds e_i - delta, e_{i+1} + delta.
bool axis_bounds(double a, double b, int K, double delta, std::vector<double> &e,
                 std::vector<double> &lo, std::vector<double> &hi) {
    const double w = (b - a) / (double)K;
    e.assign(K + 1, 0.0);
    for (int i = 0; i < K; ++i) {
        volatile double iw = (double)i * w;  // no contraction into an FMA
        e[i] = a + iw;
    }
    e[K] = b;
    for (int i = 0; i < K; ++i)
        if (!(e[i] < e[i + 1])) return false;
    lo.assign(K, 0.0);
    hi.assign(K, 0.0);
    for (int i = 0; i < K; ++i) {
        lo[i] = e[i] - delta;
        hi[i] = e[i + 1] + delta;
    }
    hi[K - 1] = std::numeric_limits<double>::infinity();
    return true;
}

}  // namespace

struct pgpcv_ctx {
    int device = 0;
    int sms = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    cudaMemPool_t pool = nullptr;  // partition scratch; keeps its memory between calls
    std::string err;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t ev_sync = nullptr;  // completion polling of collectives (no timing)

    // partition state
    bool has_partition = false;
    int64_t n = 0, N = 0;
    DevBuf<double> px, py, pv;
    DevBuf<uint8_t> prole;
    DevBuf<double> bounds;  // ex, lox, hix, ey, loy, hiy
    DevBuf<double> rects, split;      // subset rectangles [N*4]; bisection split per node id
    std::vector<double> h_rects;
    pgpcv_rect domain{};
    DevBuf<int64_t> train_off2;       // shell-cap output (swapped in)
    DevBuf<int32_t> train_idx2;
    DevBuf<unsigned int> cnt, cur;
    DevBuf<unsigned long long> stats;
    DevBuf<int64_t> train_off, val_off, test_off;
    DevBuf<int32_t> train_idx, val_idx, test_idx;
    DevBuf<uint32_t> bitmap;
    DevBuf<double> tx, ty, tv, vx, vy, vv, gx, gy, gv;  // g*: staged test points
    std::vector<int64_t> h_train_off, h_val_off, h_test_off;
    pgpcv_partition_info info{};

    // sharding
    int rank = 0, world = 1;
    ncclComm_t comm = nullptr;
    bool comm_aborted = false;  // a collective failed or timed out: shard again
    double nccl_timeout_s = 1800.0;
    DevBuf<int32_t> errflag;    // rank-local error flag for the lockstep all-reduce
    bool cv_done = false;
    std::vector<uint8_t> owned;

    // cv_loss buffers
    DevBuf<double> work;
    // per-range covariance reuse (small kernel): the blocks, per-subset offsets, the call's
    // small subsets, distinct ranges and each unique config's range index
    DevBuf<double> sig, sig_ranges;
    DevBuf<int64_t> sig_off;
    DevBuf<int32_t> sig_subs, sig_range;
    uint64_t partition_gen = 0;        // bumped by every partition (invalidates the cached layout)
    std::vector<int32_t> h_sig_subs;   // the device copies' host image (layout cache)
    std::vector<int64_t> h_sig_off;
    uint64_t sig_gen = ~0ull;          // partition_gen of the uploaded layout
    size_t sig_layout_stride = 0;
    DevBuf<double> params;
    DevBuf<int2> items;
    DevBuf<unsigned long long> counter;
    DevBuf<double> subset_loss, subset_nll, sums;  // sums: [loss C | nll C]
    DevBuf<uint8_t> fail;
    // per-unique-(range, lambda) kernel outputs (zeta dedup), expanded to the C configs
    DevBuf<double> u_loss, u_logdet, u_zz;
    DevBuf<uint8_t> u_fail;
    DevBuf<int32_t> u_map;
    DevBuf<double> u_sigma2;
    DevBuf<uint8_t> own_mask;  // [N] subsets this rank evaluated in the last call
    DevBuf<int32_t> status;                        // [loss C | nll C]
    // pgpcv_predict
    DevBuf<double> p_sub, p_yhat, p_sum;
    DevBuf<uint8_t> p_fail;
    DevBuf<int32_t> p_status;
    // pgpcv_gls
    DevBuf<double> g_X, g_tX, g_part, g_sums, g_beta;
    DevBuf<unsigned long long> prof, prof2;  // diagnostic phase cycles (-DPGPCV_PHASE_PROFILE)
    DevBuf<unsigned long long> tl;    // diagnostic timeline (-DPGPCV_TIMELINE)
    // pgpcv_select: the last evaluation's device-resident per-subset losses
    int32_t sel_C = 0;
    DevBuf<double> sel_rmspe, sel_local;
    DevBuf<int32_t> sel_best, sel_wins;
    int blocks_per_sm[kCvVariants] = {};  // resident CTAs per SM of each kernel variant
    int64_t small_k = 2048;         // subsets with k <= small_k run on the small kernel (PGPCV_SMALL_K)
    int ws = 0;                     // large kernel: the warp-specialised variant (PGPCV_WS=1)
    int sigma_reuse = 1;            // small kernel: per-range covariance blocks (PGPCV_SIGMA_REUSE: 0 never,
                                    // 1 where a subset has >= 1.5 items per range in the call, 2 always)
    double sigma_budget = 0.5;      // at most this fraction of the free device memory for the blocks
    int border_pred = 1;            // small kernel: bordered prediction where m <= k/20 (PGPCV_BORDER_PRED:
                                    // 0 never, 2 always)
    cudaStream_t aux_stream = nullptr;  // the small kernel's stream when both kernels run
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int sched = 0;  // CvArgs::sched; PGPCV_SCHED overrides (diagnostics)
    pgpcv_timing timing{};
    bool has_timing = false;

    int fail_with(int code, const char *fmt, ...) {
        char buf[1024];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        err = buf;
        return code;
    }
    int cuda_fail(cudaError_t e, const char *what) {
        cudaGetLastError();
        return fail_with(e == cudaErrorMemoryAllocation ? PGPCV_ENOMEM : PGPCV_ECUDA,
                         "%s: %s", what, cudaGetErrorString(e));
    }
};

#define CK(call, what)                                                     \
    do {                                                                   \
        cudaError_t e_ = (call);                                           \
        if (e_ != cudaSuccess) return ctx->cuda_fail(e_, what);            \
    } while (0)

namespace {

// Ownership of the subsets a call evaluates (`work[s]` != 0): LPT on k_s^3 over exactly
// those subsets (the rule documented at pgpcv_lpt_assign), so every mode balances the
// factorizations it actually runs (the likelihood and GLS factor subsets without
// validation data too).  A pure function of the partition and the call's mode, hence
// identical on every rank.  World 1 owns everything.
void assign_owned(pgpcv_ctx *ctx, const std::vector<uint8_t> &work) {
    ctx->owned.assign(ctx->N, 1);
    if (ctx->world <= 1) return;
    std::vector<int64_t> ids;
    std::vector<double> cost;
    for (int64_t s = 0; s < ctx->N; ++s) {
        if (!work[s]) continue;
        const double k = (double)(ctx->h_train_off[s + 1] - ctx->h_train_off[s]);
        ids.push_back(s);
        cost.push_back(k * k * k);
    }
    std::vector<int32_t> owner(ids.size());
    pgpcv_lpt_assign((int64_t)ids.size(), cost.data(), ctx->world, owner.data());
    for (int64_t s = 0; s < ctx->N; ++s) ctx->owned[s] = 0;
    for (size_t i = 0; i < ids.size(); ++i) ctx->owned[ids[i]] = owner[i] == ctx->rank;
}

void reset_shard(pgpcv_ctx *ctx) {
    ctx->rank = 0;
    ctx->world = 1;
    ctx->comm = nullptr;
}

// How the subsets are formed: equal tiles (R1) or the recursive bisection (row f2).
struct PartSpec {
    int kind = 0;  // 0 grid, 1 bisection
    int32_t kx = 1, ky = 1, depth = 0;
    double delta = 0;
    int64_t shell_cap = -1;  // < 0: no cap
    uint64_t seed = 0;
};

int partition_impl(pgpcv_ctx *ctx, int64_t n, const double *x, const double *y, const double *v,
                   const uint8_t *role, pgpcv_rect d, const PartSpec &ps, pgpcv_partition_info *info_out) {
    cudaStream_t st = ctx->stream;
    const double delta = ps.delta;
    ctx->has_partition = false;
    // K0: input validation on the device (NaN/Inf, outside D, bad role)
    CK(ctx->stats.ensure(3), "alloc stats");
    CK(cudaMemsetAsync(ctx->stats.p, 0, 3 * sizeof(unsigned long long), st), "memset");
    CK(launch_validate(n, x, y, v, role, d.xmin, d.xmax, d.ymin, d.ymax, ctx->stats.p, st),
       "validate kernel");
    unsigned long long hstats[3] = {0, 0, 0};
    CK(cudaMemcpyAsync(hstats, ctx->stats.p, sizeof hstats, cudaMemcpyDeviceToHost, st), "copy");
    CK(cudaStreamSynchronize(st), "validate");
    const unsigned long long flags = hstats[0];
    if (flags & 1u) return ctx->fail_with(PGPCV_EINVAL, "NaN or Inf in x, y or value");
    if (flags & 2u) return ctx->fail_with(PGPCV_EINVAL, "a point lies outside the domain");
    if (flags & 4u) return ctx->fail_with(PGPCV_EINVAL, "role byte not in {0,1,2}");

    Geom geom{};
    int64_t N = 0;
    if (ps.kind == 0) {
        const int32_t kx = ps.kx, ky = ps.ky;
        std::vector<double> ex, lox, hix, ey, loy, hiy;
        if (!axis_bounds(d.xmin, d.xmax, kx, delta, ex, lox, hix) ||
            !axis_bounds(d.ymin, d.ymax, ky, delta, ey, loy, hiy))
            return ctx->fail_with(PGPCV_EINVAL, "tile edges are not strictly increasing");
        std::vector<double> hb;
        for (auto *vec : {&ex, &lox, &hix, &ey, &loy, &hiy}) hb.insert(hb.end(), vec->begin(), vec->end());
        CK(ctx->bounds.ensure(hb.size()), "alloc bounds");
        CK(cudaMemcpyAsync(ctx->bounds.p, hb.data(), sizeof(double) * hb.size(), cudaMemcpyHostToDevice, st),
           "copy bounds");
        double *b = ctx->bounds.p;
        double *b2 = b + (kx + 1) + 2 * kx;
        geom.kind = 0;
        geom.ax = Axis{b, b + (kx + 1), b + (kx + 1) + kx, kx};
        geom.ay = Axis{b2, b2 + (ky + 1), b2 + (ky + 1) + ky, ky};
        N = (int64_t)kx * ky;
        ctx->h_rects.resize(4 * N);  // tile s = iy*kx + ix is [e_ix, e_ix+1) x [e_iy, e_iy+1)
        for (int32_t iy = 0; iy < ky; ++iy)
            for (int32_t ix = 0; ix < kx; ++ix) {
                double *r = &ctx->h_rects[4 * ((int64_t)iy * kx + ix)];
                r[0] = ex[ix];
                r[1] = ex[ix + 1];
                r[2] = ey[iy];
                r[3] = ey[iy + 1];
            }
        CK(ctx->rects.ensure(4 * N), "alloc rects");
        CK(cudaMemcpyAsync(ctx->rects.p, ctx->h_rects.data(), sizeof(double) * 4 * N, cudaMemcpyHostToDevice, st),
           "copy rects");
    } else {
        // row f2: the tree, level by level on the device (bisect.cu)
        N = (int64_t)1 << ps.depth;
        CK(ctx->split.ensure(N), "alloc split");
        CK(ctx->rects.ensure(4 * N), "alloc rects");
        CK(bisect_tree(n, x, y, role, d.xmin, d.xmax, d.ymin, d.ymax, ps.depth, delta, ctx->split.p, ctx->rects.p,
                       ctx->pool, st), "bisection");
        geom.kind = 1;
        geom.tree = Tree{ctx->split.p, ctx->rects.p, ps.depth, d.xmax, d.ymax, delta};
        ctx->h_rects.resize(4 * N);
        CK(cudaMemcpyAsync(ctx->h_rects.data(), ctx->rects.p, sizeof(double) * 4 * N, cudaMemcpyDeviceToHost, st),
           "copy rects");
    }
    ctx->N = N;
    ctx->n = n;
    ctx->domain = d;
    // K1 count, K2 scan
    CK(ctx->cnt.ensure(3 * N), "alloc counts");
    CK(ctx->cur.ensure(3 * N), "alloc cursors");
    CK(ctx->train_off.ensure(N + 1), "alloc offsets");
    CK(ctx->val_off.ensure(N + 1), "alloc offsets");
    CK(ctx->test_off.ensure(N + 1), "alloc offsets");
    CK(cudaMemsetAsync(ctx->cnt.p, 0, sizeof(unsigned) * 3 * N, st), "memset");
    CK(launch_count(n, x, y, role, geom, ctx->cnt.p, ctx->cnt.p + N, ctx->cnt.p + 2 * N, st),
       "count kernel");
    CK(launch_scan(ctx->cnt.p, N, ctx->train_off.p, st), "scan kernel");
    CK(launch_scan(ctx->cnt.p + N, N, ctx->val_off.p, st), "scan kernel");
    CK(launch_scan(ctx->cnt.p + 2 * N, N, ctx->test_off.p, st), "scan kernel");
    ctx->h_train_off.resize(N + 1);
    ctx->h_val_off.resize(N + 1);
    ctx->h_test_off.resize(N + 1);
    CK(cudaMemcpyAsync(ctx->h_train_off.data(), ctx->train_off.p, sizeof(int64_t) * (N + 1),
                       cudaMemcpyDeviceToHost, st), "copy offsets");
    CK(cudaMemcpyAsync(ctx->h_val_off.data(), ctx->val_off.p, sizeof(int64_t) * (N + 1),
                       cudaMemcpyDeviceToHost, st), "copy offsets");
    CK(cudaMemcpyAsync(ctx->h_test_off.data(), ctx->test_off.p, sizeof(int64_t) * (N + 1),
                       cudaMemcpyDeviceToHost, st), "copy offsets");
    CK(cudaStreamSynchronize(st), "scan");
    const int64_t sum_k = ctx->h_train_off[N], sum_m = ctx->h_val_off[N], sum_g = ctx->h_test_off[N];
    if (sum_k >= (int64_t)1 << 31 || sum_m >= (int64_t)1 << 31)
        return ctx->fail_with(PGPCV_EINVAL, "more than 2^31 memberships");
    // K3 scatter + per-segment sort into ascending index order
    CK(ctx->train_idx.ensure(sum_k), "alloc train_idx");
    CK(ctx->val_idx.ensure(sum_m), "alloc val_idx");
    CK(ctx->test_idx.ensure(sum_g), "alloc test_idx");
    CK(cudaMemsetAsync(ctx->cur.p, 0, sizeof(unsigned) * 3 * N, st), "memset");
    CK(launch_scatter(n, x, y, role, geom, ctx->train_off.p, ctx->val_off.p, ctx->test_off.p,
                      ctx->cur.p, ctx->cur.p + N, ctx->cur.p + 2 * N, ctx->train_idx.p,
                      ctx->val_idx.p, ctx->test_idx.p, st), "scatter kernel");
    int64_t max_k = 0, max_m = 0, max_g = 0, empty = 0;
    for (int64_t s = 0; s < N; ++s) {
        max_k = std::max(max_k, ctx->h_train_off[s + 1] - ctx->h_train_off[s]);
        const int64_t m = ctx->h_val_off[s + 1] - ctx->h_val_off[s];
        max_m = std::max(max_m, m);
        max_g = std::max(max_g, ctx->h_test_off[s + 1] - ctx->h_test_off[s]);
        empty += m == 0;
    }
    CK(launch_segsort_small(ctx->train_idx.p, ctx->train_off.p, N, max_k, st), "segsort");
    CK(launch_segsort_small(ctx->val_idx.p, ctx->val_off.p, N, max_m, st), "segsort");
    CK(launch_segsort_small(ctx->test_idx.p, ctx->test_off.p, N, max_g, st), "segsort");
    for (int which = 0; which < 3; ++which) {
        const std::vector<int64_t> &off = which == 2 ? ctx->h_test_off : which ? ctx->h_val_off : ctx->h_train_off;
        int32_t *idx = which == 2 ? ctx->test_idx.p : which ? ctx->val_idx.p : ctx->train_idx.p;
        for (int64_t s = 0; s < N; ++s) {
            const int64_t len = off[s + 1] - off[s];
            if (len > kSmallSortMax) {
                CK(ctx->bitmap.ensure((n + 31) / 32), "alloc bitmap");
                CK(sort_long_segment(idx, off[s], len, n, ctx->bitmap.p, st), "long sort");
            }
        }
    }
    // row f2: shell cap (R22) on the sorted training lists
    int64_t dropped = 0;
    if (ps.shell_cap >= 0) {
        CK(ctx->train_idx2.ensure(std::max<int64_t>(sum_k, 1)), "alloc");
        CK(ctx->train_off2.ensure(N + 1), "alloc");
        CK(cap_shells(N, ctx->train_off.p, ctx->train_idx.p, x, y, ctx->rects.p, d.xmax, d.ymax, ps.shell_cap,
                      ps.seed, ctx->train_idx2.p, ctx->train_off2.p, &dropped, ctx->pool, st), "shell cap");
        ctx->train_idx.swap(ctx->train_idx2);
        ctx->train_off.swap(ctx->train_off2);
        CK(cudaMemcpyAsync(ctx->h_train_off.data(), ctx->train_off.p, sizeof(int64_t) * (N + 1),
                           cudaMemcpyDeviceToHost, st), "copy offsets");
        CK(cudaStreamSynchronize(st), "shell cap");
        max_k = 0;
        for (int64_t s = 0; s < N; ++s) max_k = std::max(max_k, ctx->h_train_off[s + 1] - ctx->h_train_off[s]);
    }
    const int64_t sum_k_final = sum_k - dropped;
    // K4 staging gather (subset-contiguous SoA)
    CK(ctx->tx.ensure(sum_k_final), "alloc");
    CK(ctx->ty.ensure(sum_k_final), "alloc");
    CK(ctx->tv.ensure(sum_k_final), "alloc");
    CK(ctx->vx.ensure(sum_m), "alloc");
    CK(ctx->vy.ensure(sum_m), "alloc");
    CK(ctx->vv.ensure(sum_m), "alloc");
    CK(ctx->gx.ensure(sum_g), "alloc");
    CK(ctx->gy.ensure(sum_g), "alloc");
    CK(ctx->gv.ensure(sum_g), "alloc");
    CK(launch_gather(sum_k_final, ctx->train_idx.p, x, y, v, ctx->tx.p, ctx->ty.p, ctx->tv.p, st), "gather");
    CK(launch_gather(sum_m, ctx->val_idx.p, x, y, v, ctx->vx.p, ctx->vy.p, ctx->vv.p, st), "gather");
    CK(launch_gather(sum_g, ctx->test_idx.p, x, y, v, ctx->gx.p, ctx->gy.p, ctx->gv.p, st), "gather");
    CK(cudaStreamSynchronize(st), "partition");

    pgpcv_partition_info &info = ctx->info;
    info.n_subsets = N;
    info.sum_k = sum_k_final;
    info.sum_m = sum_m;
    info.max_k = max_k;
    info.max_m = max_m;
    info.n_empty_val = empty;
    info.n_train = (int64_t)hstats[1];
    info.n_val = (int64_t)hstats[2];
    info.n_test = sum_g;
    info.max_test = max_g;
    ctx->has_partition = true;
    ++ctx->partition_gen;
    ctx->cv_done = false;
    ctx->sel_C = 0;
    ctx->owned.assign(N, 1);  // each evaluation assigns its own work (assign_owned)
    if (info_out) *info_out = info;
    return PGPCV_OK;
}

}  // namespace

extern "C" {

int pgpcv_version(void) { return PGPCV_VERSION; }

int pgpcv_create(int cuda_device, pgpcv_ctx **out) {
    if (!out || cuda_device < 0) {
        g_create_error = "bad argument";
        return PGPCV_EINVAL;
    }
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        g_create_error = std::string("no CUDA device: ") + cudaGetErrorString(e);
        return PGPCV_ECUDA;
    }
    if (cuda_device >= count) {
        g_create_error = "device index out of range";
        return PGPCV_EINVAL;
    }
    cudaDeviceProp prop;
    if ((e = cudaGetDeviceProperties(&prop, cuda_device)) != cudaSuccess) {
        g_create_error = cudaGetErrorString(e);
        return PGPCV_ECUDA;
    }
    if (prop.major != 10 || prop.minor != 0) {
        g_create_error = "libpgpcv is built for sm_100a (B200) only; found compute capability " +
                         std::to_string(prop.major) + "." + std::to_string(prop.minor);
        return PGPCV_ECUDA;
    }
    pgpcv_ctx *ctx = new (std::nothrow) pgpcv_ctx();
    if (!ctx) return PGPCV_ENOMEM;
    ctx->device = cuda_device;
    ctx->sms = prop.multiProcessorCount;
    cudaSetDevice(cuda_device);
    if ((e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking)) != cudaSuccess) {
        g_create_error = cudaGetErrorString(e);
        delete ctx;
        return PGPCV_ECUDA;
    }
    ctx->stream = ctx->own_stream;
    {  // a private stream-ordered pool that never returns memory at synchronisation
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = cuda_device;
        if (cudaMemPoolCreate(&ctx->pool, &props) == cudaSuccess) {
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &keep);
        } else {
            ctx->pool = nullptr;  // fall back to the device's default pool
            cudaGetLastError();
        }
    }
    if (const char *env = getenv("PGPCV_SCHED")) ctx->sched = atoi(env);
    for (auto &ev : ctx->ev) cudaEventCreate(&ev);
    cudaEventCreateWithFlags(&ctx->ev_sync, cudaEventDisableTiming);
    for (int v = 0; v < kCvVariants; ++v)
        if ((e = cv_kernel_occupancy(v, &ctx->blocks_per_sm[v])) != cudaSuccess || ctx->blocks_per_sm[v] < 1) {
            g_create_error = std::string("cv kernel cannot be resident: ") + cudaGetErrorString(e);
            pgpcv_destroy(ctx);
            return PGPCV_ECUDA;
        }
    if ((e = cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking)) != cudaSuccess) {
        g_create_error = cudaGetErrorString(e);
        pgpcv_destroy(ctx);
        return PGPCV_ECUDA;
    }
    cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming);
    if (const char *env = getenv("PGPCV_SMALL_K")) ctx->small_k = atoll(env);
    if (const char *env = getenv("PGPCV_BORDER_PRED")) ctx->border_pred = atoi(env);
    if (const char *env = getenv("PGPCV_SIGMA_REUSE")) ctx->sigma_reuse = atoi(env);
    if (const char *env = getenv("PGPCV_WS")) ctx->ws = atoi(env);
    *out = ctx;
    return PGPCV_OK;
}

void pgpcv_destroy(pgpcv_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->comm && nccl().ok) nccl().commDestroy(ctx->comm);
    for (auto &ev : ctx->ev)
        if (ev) cudaEventDestroy(ev);
    if (ctx->ev_sync) cudaEventDestroy(ctx->ev_sync);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    if (ctx->aux_stream) cudaStreamDestroy(ctx->aux_stream);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    if (ctx->pool) cudaMemPoolDestroy(ctx->pool);
    delete ctx;
}

const char *pgpcv_last_error(const pgpcv_ctx *ctx) {
    return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

int pgpcv_set_stream(pgpcv_ctx *ctx, void *stream) {
    if (!ctx) return PGPCV_EINVAL;
    ctx->stream = stream ? (cudaStream_t)stream : ctx->own_stream;
    return PGPCV_OK;
}

static int check_partition_args(pgpcv_ctx *ctx, int64_t n, const void *x, const void *y,
                                const void *v, const void *role, pgpcv_rect d, int32_t kx,
                                int32_t ky, double delta) {
    if (n < 0 || n >= ((int64_t)1 << 31))
        return ctx->fail_with(PGPCV_EINVAL, "n must be in [0, 2^31)");
    if (n > 0 && (!x || !y || !v || !role)) return ctx->fail_with(PGPCV_EINVAL, "NULL input array");
    if (kx < 1 || ky < 1) return ctx->fail_with(PGPCV_EINVAL, "kx and ky must be >= 1");
    if ((int64_t)kx * ky > 50000000) return ctx->fail_with(PGPCV_EINVAL, "too many subsets");
    if (!(delta >= 0.0) || !std::isfinite(delta))
        return ctx->fail_with(PGPCV_EINVAL, "delta must be finite and >= 0");
    if (!(d.xmin < d.xmax) || !(d.ymin < d.ymax) || !std::isfinite(d.xmin) || !std::isfinite(d.xmax) ||
        !std::isfinite(d.ymin) || !std::isfinite(d.ymax))
        return ctx->fail_with(PGPCV_EINVAL, "invalid domain");
    return PGPCV_OK;
}

int pgpcv_partition(pgpcv_ctx *ctx, int64_t n, const double *x, const double *y, const double *value,
                    const uint8_t *role, pgpcv_rect domain, int32_t kx, int32_t ky, double delta,
                    pgpcv_partition_info *info_out) {
    NvtxRange nvtx_("pgpcv_partition");
    if (!ctx) return PGPCV_EINVAL;
    int rc = check_partition_args(ctx, n, x, y, value, role, domain, kx, ky, delta);
    if (rc) return rc;
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    CK(ctx->px.ensure(n), "alloc points");
    CK(ctx->py.ensure(n), "alloc points");
    CK(ctx->pv.ensure(n), "alloc points");
    CK(ctx->prole.ensure(n), "alloc points");
    if (n > 0) {
        CK(cudaMemcpyAsync(ctx->px.p, x, sizeof(double) * n, cudaMemcpyHostToDevice, st), "copy x");
        CK(cudaMemcpyAsync(ctx->py.p, y, sizeof(double) * n, cudaMemcpyHostToDevice, st), "copy y");
        CK(cudaMemcpyAsync(ctx->pv.p, value, sizeof(double) * n, cudaMemcpyHostToDevice, st), "copy v");
        CK(cudaMemcpyAsync(ctx->prole.p, role, n, cudaMemcpyHostToDevice, st), "copy role");
    }
    PartSpec ps;
    ps.kx = kx;
    ps.ky = ky;
    ps.delta = delta;
    return partition_impl(ctx, n, ctx->px.p, ctx->py.p, ctx->pv.p, ctx->prole.p, domain, ps, info_out);
}

int pgpcv_partition_device(pgpcv_ctx *ctx, int64_t n, const double *d_x, const double *d_y,
                           const double *d_value, const uint8_t *d_role, pgpcv_rect domain,
                           int32_t kx, int32_t ky, double delta, pgpcv_partition_info *info_out) {
    NvtxRange nvtx_("pgpcv_partition_device");
    if (!ctx) return PGPCV_EINVAL;
    int rc = check_partition_args(ctx, n, d_x, d_y, d_value, d_role, domain, kx, ky, delta);
    if (rc) return rc;
    cudaSetDevice(ctx->device);
    PartSpec ps;
    ps.kx = kx;
    ps.ky = ky;
    ps.delta = delta;
    return partition_impl(ctx, n, d_x, d_y, d_value, d_role, domain, ps, info_out);
}

static int bisect_spec(pgpcv_ctx *ctx, int32_t depth, double delta, int64_t shell_cap, uint64_t seed, PartSpec &ps) {
    if (depth < 0 || depth > 20) return ctx->fail_with(PGPCV_EINVAL, "depth must be in [0, 20]");
    ps.kind = 1;
    ps.depth = depth;
    ps.delta = delta;
    ps.shell_cap = shell_cap;
    ps.seed = seed;
    return PGPCV_OK;
}

int pgpcv_partition_bisect(pgpcv_ctx *ctx, int64_t n, const double *x, const double *y, const double *value,
                           const uint8_t *role, pgpcv_rect domain, int32_t depth, double delta, int64_t shell_cap,
                           uint64_t seed, pgpcv_partition_info *info_out) {
    NvtxRange nvtx_("pgpcv_partition_bisect");
    if (!ctx) return PGPCV_EINVAL;
    int rc = check_partition_args(ctx, n, x, y, value, role, domain, 1, 1, delta);
    if (rc) return rc;
    PartSpec ps;
    if ((rc = bisect_spec(ctx, depth, delta, shell_cap, seed, ps))) return rc;
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    CK(ctx->px.ensure(n), "alloc points");
    CK(ctx->py.ensure(n), "alloc points");
    CK(ctx->pv.ensure(n), "alloc points");
    CK(ctx->prole.ensure(n), "alloc points");
    if (n > 0) {
        CK(cudaMemcpyAsync(ctx->px.p, x, sizeof(double) * n, cudaMemcpyHostToDevice, st), "copy x");
        CK(cudaMemcpyAsync(ctx->py.p, y, sizeof(double) * n, cudaMemcpyHostToDevice, st), "copy y");
        CK(cudaMemcpyAsync(ctx->pv.p, value, sizeof(double) * n, cudaMemcpyHostToDevice, st), "copy v");
        CK(cudaMemcpyAsync(ctx->prole.p, role, n, cudaMemcpyHostToDevice, st), "copy role");
    }
    return partition_impl(ctx, n, ctx->px.p, ctx->py.p, ctx->pv.p, ctx->prole.p, domain, ps, info_out);
}

int pgpcv_partition_bisect_device(pgpcv_ctx *ctx, int64_t n, const double *d_x, const double *d_y,
                                  const double *d_value, const uint8_t *d_role, pgpcv_rect domain, int32_t depth,
                                  double delta, int64_t shell_cap, uint64_t seed, pgpcv_partition_info *info_out) {
    NvtxRange nvtx_("pgpcv_partition_bisect_device");
    if (!ctx) return PGPCV_EINVAL;
    int rc = check_partition_args(ctx, n, d_x, d_y, d_value, d_role, domain, 1, 1, delta);
    if (rc) return rc;
    PartSpec ps;
    if ((rc = bisect_spec(ctx, depth, delta, shell_cap, seed, ps))) return rc;
    cudaSetDevice(ctx->device);
    return partition_impl(ctx, n, d_x, d_y, d_value, d_role, domain, ps, info_out);
}

int pgpcv_partition_rects(pgpcv_ctx *ctx, double *rects) {
    if (!ctx || !rects) return PGPCV_EINVAL;
    if (!ctx->has_partition) return ctx->fail_with(PGPCV_ESTATE, "no partition");
    memcpy(rects, ctx->h_rects.data(), sizeof(double) * ctx->h_rects.size());
    return PGPCV_OK;
}

int pgpcv_partition_export(pgpcv_ctx *ctx, int64_t *train_off, int32_t *train_idx, int64_t *val_off,
                           int32_t *val_idx) {
    if (!ctx) return PGPCV_EINVAL;
    if (!ctx->has_partition) return ctx->fail_with(PGPCV_ESTATE, "no partition");
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    const int64_t N = ctx->N;
    if (train_off) memcpy(train_off, ctx->h_train_off.data(), sizeof(int64_t) * (N + 1));
    if (val_off) memcpy(val_off, ctx->h_val_off.data(), sizeof(int64_t) * (N + 1));
    if (train_idx && ctx->info.sum_k)
        CK(cudaMemcpyAsync(train_idx, ctx->train_idx.p, sizeof(int32_t) * ctx->info.sum_k,
                           cudaMemcpyDeviceToHost, st), "copy train_idx");
    if (val_idx && ctx->info.sum_m)
        CK(cudaMemcpyAsync(val_idx, ctx->val_idx.p, sizeof(int32_t) * ctx->info.sum_m,
                           cudaMemcpyDeviceToHost, st), "copy val_idx");
    CK(cudaStreamSynchronize(st), "export");
    return PGPCV_OK;
}

int pgpcv_nccl_get_unique_id(void *out) {
    if (!out) return PGPCV_EINVAL;
    NcclApi &api = nccl();
    if (!api.ok) return PGPCV_ENCCL;
    ncclUniqueId id;
    if (api.getUniqueId(&id) != ncclSuccess) return PGPCV_ENCCL;
    memcpy(out, &id, sizeof id);
    return PGPCV_OK;
}

int pgpcv_shard(pgpcv_ctx *ctx, int rank, int world, const void *nccl_unique_id) {
    NvtxRange nvtx_("pgpcv_shard");
    if (!ctx) return PGPCV_EINVAL;
    if (world < 1 || rank < 0 || rank >= world)
        return ctx->fail_with(PGPCV_EINVAL, "need 0 <= rank < world");
    if (!ctx->has_partition) return ctx->fail_with(PGPCV_ESTATE, "pgpcv_shard needs a partition");
    if (ctx->cv_done && !ctx->comm_aborted)
        return ctx->fail_with(PGPCV_ESTATE, "pgpcv_shard after pgpcv_cv_loss on this partition");
    // Validate every prerequisite before touching the ctx's sharding state: a failed call
    // leaves the ctx at rank 0 of world 1 (it then owns every subset and runs no collective).
    NcclApi *api = nullptr;
    if (world > 1) {
        if (!nccl_unique_id) return ctx->fail_with(PGPCV_EINVAL, "world > 1 needs an ncclUniqueId");
        api = &nccl();
        if (!api->ok) return ctx->fail_with(PGPCV_ENCCL, "%s", api->why.c_str());
    }
    cudaSetDevice(ctx->device);
    if (ctx->comm) {
        nccl().commDestroy(ctx->comm);
        ctx->comm = nullptr;
    }
    reset_shard(ctx);
    ctx->comm_aborted = false;
    if (world > 1) {
        ncclUniqueId id;
        memcpy(&id, nccl_unique_id, sizeof id);
        ncclComm_t comm = nullptr;
        ncclResult_t r = api->commInitRank(&comm, world, id, rank);
        if (r != ncclSuccess) return ctx->fail_with(PGPCV_ENCCL, "ncclCommInitRank: %s", api->getErrorString(r));
        ctx->comm = comm;
        ctx->rank = rank;
        ctx->world = world;
    }
    if (const char *env = getenv("PGPCV_NCCL_TIMEOUT_S")) ctx->nccl_timeout_s = atof(env);
    return PGPCV_OK;
}

int pgpcv_nccl_library(char *buf, int64_t len) {
    if (!buf || len < 1) return PGPCV_EINVAL;
    NcclApi &api = nccl();
    snprintf(buf, (size_t)len, "%s", api.where.c_str());
    return api.ok ? PGPCV_OK : PGPCV_ENCCL;
}

}  // extern "C"

namespace {

int check_params(pgpcv_ctx *ctx, const pgpcv_param *params, int32_t n_params) {
    if (n_params < 1 || !params) return ctx->fail_with(PGPCV_EINVAL, "need n_params >= 1 configurations");
    for (int c = 0; c < n_params; ++c) {
        const pgpcv_param &p = params[c];
        if (!(p.range > 0) || !(p.sigma2 > 0) || !(p.nugget >= 0) || !std::isfinite(p.range) ||
            !std::isfinite(p.sigma2) || !std::isfinite(p.nugget))
            return ctx->fail_with(PGPCV_EINVAL, "config %d: need range > 0, sigma2 > 0, nugget >= 0", c);
    }
    return PGPCV_OK;
}

// One launch of the batched CV kernel over `items` (subset, config) in LPT order, with the
// factor workspace sized for the largest subset; records the launch's CUDA-event time on
// ctx->ev[1..2].  Outputs are device arrays of stride out_C (see CvArgs).
struct CvLaunch {
    int32_t flags = 0;
    const pgpcv_param *params = nullptr;
    int32_t C = 0;
    std::vector<int2> items;
    int32_t out_C = 1;
    const int64_t *tgt_off = nullptr;   // device target offsets
    const int64_t *h_tgt_off = nullptr; // the same offsets on the host
    const double *gx = nullptr, *gy = nullptr, *gv = nullptr;
    double *subset_loss = nullptr, *logdet = nullptr, *zz = nullptr, *yhat = nullptr;
    uint8_t *fail = nullptr;
    int launches = 0;  // kernel launches run_cv made
    int32_t p = 0;  // GLS covariates (bordered rows below y)
    const double *tX = nullptr;
    double *gls_out = nullptr;
    double flops = 0;
    int slots = 0;
};

uint64_t dbits(double v) {
    uint64_t u;
    memcpy(&u, &v, sizeof u);
    return u;
}

// One batched evaluation of `items` (subset, config) in LPT order (descending k): items
// with k > small_k run on the large-subset kernel, the rest on the small-subset kernel
// (cv_kernel.cu, Geo<128,64,2> / Geo<64,32,4>), the two launched on forked streams so the
// small kernel's CTAs fill SMs as the large kernel's persistent CTAs drain.  Each kernel
// gets one factor slot per resident CTA, sized for its largest subset.  Records the span
// of the launches on ctx->ev[1..2].  Outputs are device arrays of stride out_C (CvArgs).
int run_cv(pgpcv_ctx *ctx, CvLaunch &L) {
    NvtxRange nvtx_("run_cv");
    cudaStream_t st = ctx->stream;
    auto kof = [&](const int2 &it) { return ctx->h_train_off[it.x + 1] - ctx->h_train_off[it.x]; };
    // LPT: descending k (stable, so ties keep ascending subset / config order)
    std::stable_sort(L.items.begin(), L.items.end(), [&](const int2 &a, const int2 &b) { return kof(a) > kof(b); });
    int64_t kmax = 0;
    for (const int2 &it : L.items) kmax = std::max(kmax, kof(it));
    if (kmax > cv_kernel_max_k())
        return ctx->fail_with(PGPCV_EINVAL, "a subset has %lld training points (max %d)", (long long)kmax,
                              cv_kernel_max_k());
    const int64_t n_items = (int64_t)L.items.size();
    if (n_items >= ((int64_t)1 << 31)) return ctx->fail_with(PGPCV_EINVAL, "too many work items");
    // split point: items [0, n_large) are large, [n_large, n_items) small
    int64_t n_large = 0;
    while (n_large < n_items && kof(L.items[n_large]) > ctx->small_k) ++n_large;
    struct Part {
        int variant;
        int64_t first, count, kmax;
        int slots = 0;
        size_t stride = 0, offset = 0;
        int border = 0;    // bordered prediction (targets as extra factor rows)
        int64_t extra = 0; // bordered rows below y: covariates (GLS) or targets
    } parts[2] = {{ctx->ws ? kCvLargeWS : kCvLarge, 0, n_large, n_large ? kof(L.items[0]) : 0},
                  {kCvSmall, n_large, n_items - n_large, n_items > n_large ? kof(L.items[n_large]) : 0}};
    // The small kernel predicts by bordering the targets below y (one factorization sweep,
    // no back-substitution: DESIGN.md section 6) -- m k^2 extra DMMA flops, against a
    // latency-bound re-read of the whole factor; the large kernel back-substitutes.
    for (Part &q : parts) {
        q.extra = L.p;
        q.border = ((L.flags & kCvPredict) && q.variant != kCvLarge) ? ctx->border_pred : 0;
        if (q.border)
            for (int64_t i = q.first; i < q.first + q.count; ++i) {
                const int s = L.items[i].x;
                q.extra = std::max<int64_t>(q.extra, L.h_tgt_off[s + 1] - L.h_tgt_off[s]);
            }
    }
    std::vector<double> hp(3 * (size_t)L.C);
    for (int c = 0; c < L.C; ++c) {
        hp[3 * c] = L.params[c].range;
        hp[3 * c + 1] = L.params[c].sigma2;
        hp[3 * c + 2] = L.params[c].nugget;
    }
    CK(ctx->params.ensure(3 * (size_t)L.C), "alloc params");
    CK(ctx->items.ensure(std::max<int64_t>(n_items, 1)), "alloc items");
    CK(ctx->counter.ensure(2 * (1 + kMaxSms)), "alloc counter");
    // factor workspace: one factor per resident CTA of each kernel
    int cap = 0;
    if (const char *env = getenv("PGPCV_MAX_SLOTS")) cap = atoi(env);  // diagnostics: cap resident CTAs
    size_t total = 0;
    for (Part &q : parts) {
        if (!q.count) continue;
        q.slots = (int)std::min<int64_t>((int64_t)ctx->sms * ctx->blocks_per_sm[q.variant], q.count);
        if (cap > 0) q.slots = std::min(q.slots, cap);
        const int per_cta = cv_kernel_slots_per_cta(q.variant);  // WS: two item streams per CTA
        q.slots = (q.slots + per_cta - 1) / per_cta * per_cta;
        q.stride = cv_kernel_slot_doubles(q.variant, q.kmax, (int)q.extra);
    }
    while (true) {
        total = 0;
        for (Part &q : parts) {
            q.offset = total;
            total += (size_t)q.slots * q.stride;
        }
        cudaError_t e = ctx->work.ensure(std::max<size_t>(total, 1));
        if (e == cudaSuccess) break;
        Part &big = parts[0].slots * parts[0].stride >= parts[1].slots * parts[1].stride ? parts[0] : parts[1];
        if (big.slots <= 1) return ctx->cuda_fail(e, "alloc factor workspace");
        big.slots = std::max(1, big.slots / 2);
    }
    L.slots = parts[0].slots + parts[1].slots;
    CK(cudaMemcpyAsync(ctx->params.p, hp.data(), sizeof(double) * hp.size(), cudaMemcpyHostToDevice, st),
       "copy params");
    if (n_items)
        CK(cudaMemcpyAsync(ctx->items.p, L.items.data(), sizeof(int2) * n_items, cudaMemcpyHostToDevice, st),
           "copy items");
    CK(cudaMemsetAsync(ctx->counter.p, 0, sizeof(unsigned long long) * 2 * (1 + kMaxSms), st), "memset");
    // Per-range covariance reuse for the small kernel (K4s): when the
    // small items outnumber the (subset, range) blocks by half again (or always with
    // PGPCV_SIGMA_REUSE=2), Sigma_theta of every small subset is generated once per range by
    // sigma_kernel and read by the items.  The blocks live for this call only (nothing is
    // cached across calls but their layout, a function of the partition); skipped when they
    // would take more than sigma_budget of the free device memory.
    bool use_sig = false;
    int32_t n_sub_small = 0, n_ranges = 0;
    size_t sig_stride = 0;
    {
        const Part &q = parts[1];
        std::vector<int32_t> range_of(L.C);
        std::vector<uint64_t> rkeys;
        std::vector<double> rvals;
        for (int c = 0; c < L.C; ++c) {
            const uint64_t key = dbits(L.params[c].range);
            int32_t r = (int32_t)(std::find(rkeys.begin(), rkeys.end(), key) - rkeys.begin());
            if (r == (int32_t)rkeys.size()) {
                rkeys.push_back(key);
                rvals.push_back(L.params[c].range);
            }
            range_of[c] = r;
        }
        n_ranges = (int32_t)rkeys.size();
        if (q.count && ctx->sigma_reuse > 0) {
            std::vector<int32_t> subs;
            std::vector<int64_t> off(ctx->N, -1);
            size_t total_sig = 0;
            for (int64_t i = q.first; i < q.first + q.count; ++i) {
                const int s = L.items[i].x;
                if (off[s] >= 0) continue;
                const int64_t k = kof(L.items[i]), m = L.h_tgt_off[s + 1] - L.h_tgt_off[s];
                off[s] = (int64_t)total_sig;
                subs.push_back(s);
                total_sig += (size_t)(sigma_doubles(k, border_rows(L.flags, q.border, k, m)) + 31) / 32 * 32;
            }
            // worth it when the items outnumber the blocks generated by half again (a block
            // costs one generation; an item reading it saves one)
            const bool want = ctx->sigma_reuse == 2 || 2 * q.count >= 3 * (int64_t)subs.size() * n_ranges;
            const size_t need = total_sig * (size_t)n_ranges;
            bool fits = want && need > 0 && need <= ctx->sig.cap;
            if (want && need > 0 && !fits) {  // grow (the only place that asks for free memory)
                size_t free_b = 0, tot_b = 0;
                cudaMemGetInfo(&free_b, &tot_b);
                fits = (double)need * sizeof(double) <= ctx->sigma_budget * (double)free_b &&
                       ctx->sig.ensure(need) == cudaSuccess;
            }
            if (fits) {
                const bool same = ctx->sig_gen == ctx->partition_gen && subs == ctx->h_sig_subs && off == ctx->h_sig_off;
                if (!same) {
                    CK(ctx->sig_off.ensure(ctx->N), "alloc");
                    CK(ctx->sig_subs.ensure(subs.size()), "alloc");
                    CK(cudaMemcpyAsync(ctx->sig_off.p, off.data(), sizeof(int64_t) * ctx->N, cudaMemcpyHostToDevice,
                                       st), "copy");
                    CK(cudaMemcpyAsync(ctx->sig_subs.p, subs.data(), sizeof(int32_t) * subs.size(),
                                       cudaMemcpyHostToDevice, st), "copy");
                    ctx->h_sig_subs.swap(subs);
                    ctx->h_sig_off.swap(off);
                    ctx->sig_gen = ctx->partition_gen;
                }
                CK(ctx->sig_ranges.ensure(n_ranges), "alloc");
                CK(ctx->sig_range.ensure(L.C), "alloc");
                CK(cudaMemcpyAsync(ctx->sig_ranges.p, rvals.data(), sizeof(double) * n_ranges, cudaMemcpyHostToDevice,
                                   st), "copy");
                CK(cudaMemcpyAsync(ctx->sig_range.p, range_of.data(), sizeof(int32_t) * L.C, cudaMemcpyHostToDevice,
                                   st), "copy");
                use_sig = true;
                n_sub_small = (int32_t)ctx->h_sig_subs.size();
                sig_stride = total_sig;
            }
        }
    }
    CK(cudaEventRecord(ctx->ev[1], st), "event");
    if (use_sig) parts[1].variant = kCvSmallSig;  // same geometry, slots and SMEM as kCvSmall
    const bool both = parts[0].count && parts[1].count;
    if (both) {  // fork: the small kernel on the auxiliary stream
        CK(cudaEventRecord(ctx->ev_fork, st), "event");
        CK(cudaStreamWaitEvent(ctx->aux_stream, ctx->ev_fork, 0), "stream wait");
    }
    for (int pi = 0; pi < 2; ++pi) {
        const Part &q = parts[pi];
        if (!q.count) continue;
        cudaStream_t ls = (both && pi == 1) ? ctx->aux_stream : st;
        CvArgs a;
        a.train_off = ctx->train_off.p;
        a.val_off = L.tgt_off;
        a.tx = ctx->tx.p;
        a.ty = ctx->ty.p;
        a.tv = ctx->tv.p;
        a.vx = L.gx;
        a.vy = L.gy;
        a.vv = L.gv;
        a.params = ctx->params.p;
        a.C = L.C;
        a.items = ctx->items.p + q.first;
        a.n_items = (int32_t)q.count;
        a.counter = ctx->counter.p + pi * (1 + kMaxSms);
        a.sched = ctx->sched;
        a.work = ctx->work.p + q.offset;
        a.slot_stride = q.stride;
        a.out_C = L.out_C;
        a.flags = L.flags;
        a.border_pred = q.border;
        a.subset_loss = L.subset_loss;
        a.logdet = L.logdet;
        a.zz = L.zz;
        a.yhat = L.yhat;
        a.fail = L.fail;
        a.p = L.p;
        a.tX = L.tX;
        a.rects = ctx->rects.p;
        a.xmax = ctx->domain.xmax;
        a.ymax = ctx->domain.ymax;
        a.gls_out = L.gls_out;
        a.sig = nullptr;
        a.sig_off = nullptr;
        a.sig_stride = 0;
        a.sig_range = nullptr;
        if (pi == 1 && use_sig) {
            CK(launch_sigma(ctx->sig_subs.p, n_sub_small, ctx->sig_ranges.p, n_ranges, ctx->train_off.p, L.tgt_off,
                            ctx->tx.p, ctx->ty.p, L.gx, L.gy, L.flags, q.border, ctx->sig.p, ctx->sig_off.p,
                            sig_stride, ls), "sigma kernel launch");
            ++L.launches;
            a.sig = ctx->sig.p;
            a.sig_off = ctx->sig_off.p;
            a.sig_stride = sig_stride;
            a.sig_range = ctx->sig_range.p;
        }
        a.prof = nullptr;
#ifdef PGPCV_PHASE_PROFILE
        DevBuf<unsigned long long> &prof = pi ? ctx->prof2 : ctx->prof;
        CK(prof.ensure((size_t)q.slots * 15), "alloc prof");
        CK(cudaMemsetAsync(prof.p, 0, sizeof(unsigned long long) * q.slots * 15, ls), "memset");
        a.prof = prof.p;
#endif
        a.tl = nullptr;
#ifdef PGPCV_TIMELINE
        CK(ctx->tl.ensure((size_t)q.slots * 32768), "alloc timeline");
        CK(cudaMemsetAsync(ctx->tl.p, 0, sizeof(unsigned long long) * q.slots * 32768, ls), "memset");
        a.tl = pi == 0 ? ctx->tl.p : nullptr;  // the large kernel's timeline only
#endif
        CK(launch_cv_kernel(q.variant, a, q.slots, ls), "cv kernel launch");
        ++L.launches;
    }
    if (both) {  // join
        CK(cudaEventRecord(ctx->ev_join, ctx->aux_stream), "event");
        CK(cudaStreamWaitEvent(st, ctx->ev_join, 0), "stream wait");
    }
    CK(cudaEventRecord(ctx->ev[2], st), "event");
#ifdef PGPCV_TIMELINE
    if (const char *path = getenv("PGPCV_TIMELINE_FILE"))
        if (parts[0].count) {
            std::vector<unsigned long long> h((size_t)parts[0].slots * 32768);
            CK(cudaMemcpyAsync(h.data(), ctx->tl.p, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost,
                               st), "copy timeline");
            CK(cudaStreamSynchronize(st), "timeline");
            if (FILE *f = fopen(path, "wb")) {
                fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
                fclose(f);
            }
        }
#endif
#ifdef PGPCV_PHASE_PROFILE
    for (int pi = 0; pi < 2; ++pi) {
        const Part &q = parts[pi];
        if (!q.count) continue;
        std::vector<unsigned long long> h((size_t)q.slots * 15);
        CK(cudaMemcpyAsync(h.data(), (pi ? ctx->prof2 : ctx->prof).p, sizeof(unsigned long long) * h.size(),
                           cudaMemcpyDeviceToHost, st), "copy prof");
        CK(cudaStreamSynchronize(st), "prof");
        double sum[15] = {0};
        for (int b = 0; b < q.slots; ++b)
            for (int i = 0; i < 15; ++i) sum[i] += (double)h[(size_t)b * 15 + i];
        fprintf(stderr, "PGPCV_PHASES {\"variant\": %d, \"slots\": %d, \"cycles\": [", q.variant, q.slots);
        for (int i = 0; i < 15; ++i) fprintf(stderr, "%s%.6e", i ? ", " : "", sum[i]);
        fprintf(stderr, "]}\n");
    }
#endif
    return PGPCV_OK;
}

void record_timing(pgpcv_ctx *ctx, const CvLaunch &L, int launches, int32_t configs_executed) {
    float kms = 0, tms = 0;
    cudaEventElapsedTime(&kms, ctx->ev[1], ctx->ev[2]);
    cudaEventElapsedTime(&tms, ctx->ev[0], ctx->ev[3]);
    ctx->timing.kernel_ms = kms;
    ctx->timing.total_ms = tms;
    ctx->timing.flops = L.flops;
    ctx->timing.n_evals = (int64_t)L.items.size();
    ctx->timing.launches = launches;
    ctx->timing.n_slots = L.slots;
    ctx->timing.n_configs_executed = configs_executed;
    ctx->has_timing = true;
}

int nccl_sum(pgpcv_ctx *ctx, void *buf, size_t count, ncclDataType_t t, ncclRedOp_t op = ncclSum) {
    NcclApi &api = nccl();
    ncclResult_t r = api.allReduce(buf, buf, count, t, op, ctx->comm, ctx->stream);
    if (r != ncclSuccess) return ctx->fail_with(PGPCV_ENCCL, "ncclAllReduce: %s", api.getErrorString(r));
    return PGPCV_OK;
}

// Wait for the work enqueued on the ctx stream (collectives included) while polling the
// communicator for asynchronous errors.  An NCCL error, or no completion within
// nccl_timeout_s (a hung or dead peer), aborts the communicator: the call returns ENCCL and
// the ctx needs pgpcv_shard again before another multi-rank evaluation.
int wait_collective(pgpcv_ctx *ctx, const char *what) {
    NcclApi &api = nccl();
    CK(cudaEventRecord(ctx->ev_sync, ctx->stream), "event");
    const double t0 = now_s();
    for (long spins = 0;; ++spins) {
        const cudaError_t q = cudaEventQuery(ctx->ev_sync);
        if (q == cudaSuccess) return PGPCV_OK;
        if (q != cudaErrorNotReady) return ctx->cuda_fail(q, what);
        ncclResult_t ar = ncclSuccess;
        api.commGetAsyncError(ctx->comm, &ar);
        const bool bad = ar != ncclSuccess && ar != ncclInProgress;
        const double waited = now_s() - t0;
        if (bad || waited > ctx->nccl_timeout_s) {
            api.commAbort(ctx->comm);
            ctx->comm = nullptr;
            ctx->comm_aborted = true;
            if (bad)
                return ctx->fail_with(PGPCV_ENCCL, "%s: NCCL error %s (communicator aborted; call pgpcv_shard again)",
                                      what, api.getErrorString(ar));
            return ctx->fail_with(PGPCV_ENCCL, "%s: no completion after %.0f s (a peer hung or died; communicator "
                                  "aborted; call pgpcv_shard again)", what, waited);
        }
        if (spins < 2000)
            sched_yield();
        else
            usleep(100);
    }
}

// End of a call: world 1 synchronises the stream; world > 1 polls (wait_collective).
int finish(pgpcv_ctx *ctx, const char *what) {
    if (ctx->world > 1) {
        int rc = wait_collective(ctx, what);
        if (rc) return rc;
    } else {
        CK(cudaStreamSynchronize(ctx->stream), what);
    }
    CK(cudaGetLastError(), what);
    return PGPCV_OK;
}

// Lockstep of the ranks (world > 1): every rank arrives here after its rank-local work
// with its outcome rc (argument checks that depend on the whole partition ran before any
// rank-local work, identically on every rank).  One MAX all-reduce of the error flags
// decides for all ranks together whether the data collectives run, so no rank enqueues a
// collective that a failed peer will never join.  Returns rc, or ENCCL when a peer failed.
int join_ranks(pgpcv_ctx *ctx, int rc) {
    if (ctx->world <= 1) return rc;
    if (const char *f = getenv("PGPCV_TEST_FAIL_RANK"))  // fault injection for the lockstep test
        if (rc == PGPCV_OK && atoi(f) == ctx->rank)
            rc = ctx->fail_with(PGPCV_ENOMEM, "injected rank-local failure (PGPCV_TEST_FAIL_RANK)");
    if (rc == PGPCV_OK) {  // the local work must be complete, asynchronous errors included
        cudaError_t e = cudaStreamSynchronize(ctx->stream);
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e != cudaSuccess) rc = ctx->cuda_fail(e, "rank-local evaluation");
    }
    const std::string local_err = ctx->err;
    int32_t flag = rc ? 1 : 0;
    CK(ctx->errflag.ensure(1), "alloc");
    CK(cudaMemcpyAsync(ctx->errflag.p, &flag, sizeof flag, cudaMemcpyHostToDevice, ctx->stream), "copy flag");
    int r2 = nccl_sum(ctx, ctx->errflag.p, 1, ncclInt32, ncclMax);
    if (!r2) {
        CK(cudaMemcpyAsync(&flag, ctx->errflag.p, sizeof flag, cudaMemcpyDeviceToHost, ctx->stream), "copy flag");
        r2 = wait_collective(ctx, "error-flag all-reduce");
    }
    if (rc) {
        ctx->err = local_err;
        return rc;
    }
    if (r2) return r2;
    if (flag) return ctx->fail_with(PGPCV_ENCCL, "a peer rank failed its local evaluation");
    return PGPCV_OK;
}

// Checks that must give the same answer on every rank, before any rank-local work.
int check_common(pgpcv_ctx *ctx) {
    if (ctx->info.max_k > cv_kernel_max_k())
        return ctx->fail_with(PGPCV_EINVAL, "a subset has %lld training points (max %d)",
                              (long long)ctx->info.max_k, cv_kernel_max_k());
    if (ctx->world > 1 && !ctx->comm)
        return ctx->fail_with(PGPCV_ENCCL, "the communicator was aborted by an earlier failure; call pgpcv_shard "
                                           "again");
    return PGPCV_OK;
}

int first_fail(int32_t a, int32_t b) { return a < 0 ? b : (b < 0 ? a : std::min(a, b)); }


}  // namespace

extern "C" {

int pgpcv_evaluate(pgpcv_ctx *ctx, const pgpcv_param *params, int32_t n_params, const pgpcv_outputs *out) {
    NvtxRange nvtx_("pgpcv_evaluate");
    if (!ctx) return PGPCV_EINVAL;
    if (!ctx->has_partition) return ctx->fail_with(PGPCV_ESTATE, "evaluation needs a partition");
    if (!out) return ctx->fail_with(PGPCV_EINVAL, "NULL outputs");
    int rc = check_params(ctx, params, n_params);
    if (rc) return rc;
    const bool want_cv = out->loss || out->subset_loss;
    const bool want_nll = out->nll || out->subset_nll;
    if (!want_cv && !want_nll) return ctx->fail_with(PGPCV_EINVAL, "no output requested");
    if (want_cv && ctx->info.sum_m == 0) return ctx->fail_with(PGPCV_EEMPTY, "no subset has validation data");
    if ((rc = check_common(ctx))) return rc;
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    const int64_t N = ctx->N;
    const int32_t C = n_params;
    ctx->sel_C = 0;

    // zeta dedup (the prediction depends on zeta only through (range, lambda), lambda
    // = nugget / sigma2): configs whose (range, lambda) are bit-identical share one
    // factorization per subset.  lambda is the same IEEE division the kernel performs, so
    // the shared results are exactly those each config would compute.  Nothing is cached
    // across calls.
    std::vector<int32_t> umap(C);
    std::vector<pgpcv_param> uparams;
    std::vector<double> sig2(C);
    {
        std::vector<std::pair<uint64_t, uint64_t>> keys;
        for (int32_t c = 0; c < C; ++c) {
            const volatile double lam = params[c].nugget / params[c].sigma2;
            const std::pair<uint64_t, uint64_t> key(dbits(params[c].range), dbits(lam));
            int32_t u = (int32_t)(std::find(keys.begin(), keys.end(), key) - keys.begin());
            if (u == (int32_t)keys.size()) {
                keys.push_back(key);
                uparams.push_back(params[c]);
            }
            umap[c] = u;
            sig2[c] = params[c].sigma2;
        }
    }
    const int32_t U = (int32_t)uparams.size();

    CvLaunch L;
    L.flags = (want_cv ? kCvPredict : 0) | (want_nll ? kCvNll : 0);
    L.params = uparams.data();
    L.C = U;
    L.out_C = U;
    L.tgt_off = ctx->val_off.p;
    L.h_tgt_off = ctx->h_val_off.data();
    L.gx = ctx->vx.p;
    L.gy = ctx->vy.p;
    L.gv = ctx->vv.p;
    // subsets this call factors: those with validation data, every subset when the
    // likelihood is requested (it needs no targets); this rank's share by LPT on k^3
    std::vector<uint8_t> work(N), own(N);
    for (int64_t s = 0; s < N; ++s) work[s] = (ctx->h_val_off[s + 1] > ctx->h_val_off[s]) || want_nll;
    assign_owned(ctx, work);
    for (int64_t s = 0; s < N; ++s) {
        own[s] = work[s] && ctx->owned[s];
        if (!own[s]) continue;
        const int64_t k = ctx->h_train_off[s + 1] - ctx->h_train_off[s];
        const int64_t m = ctx->h_val_off[s + 1] - ctx->h_val_off[s];
        for (int32_t u = 0; u < U; ++u) L.items.push_back(make_int2((int)s, u));
        // the Cholesky and forward solve count for every executed item; the
        // backward solve, prediction and residuals only where validation data are predicted.
        const double kd = (double)k, md = (double)m;
        double f = kd * kd * kd / 3.0 + kd * kd / 2.0 + kd / 6.0 + kd * kd;
        if (want_cv && m > 0) f += kd * kd + 2.0 * md * kd + 3.0 * md;
        L.flops += U * f;
    }
    const bool multi = ctx->world > 1;
    const bool gather = multi && (out->subset_loss || out->subset_nll);
    int launches = 0;

    // ---- rank-local phase: factor this rank's (subset, unique config) items ----
    auto local = [&]() -> int {
        CK(ctx->subset_loss.ensure((size_t)N * C), "alloc subset_loss");
        CK(ctx->subset_nll.ensure((size_t)N * C), "alloc subset_nll");
        CK(ctx->fail.ensure((size_t)N * C), "alloc fail");
        CK(ctx->u_loss.ensure((size_t)N * U), "alloc");
        CK(ctx->u_fail.ensure((size_t)N * U), "alloc");
        CK(ctx->u_logdet.ensure(want_nll ? (size_t)N * U : 1), "alloc");
        CK(ctx->u_zz.ensure(want_nll ? (size_t)N * U : 1), "alloc");
        CK(ctx->u_map.ensure(C), "alloc");
        CK(ctx->u_sigma2.ensure(C), "alloc");
        CK(ctx->own_mask.ensure(N), "alloc");
        CK(ctx->sums.ensure(2 * (size_t)C), "alloc sums");
        CK(ctx->status.ensure(2 * (size_t)C), "alloc status");
        L.subset_loss = ctx->u_loss.p;
        L.logdet = want_nll ? ctx->u_logdet.p : nullptr;
        L.zz = want_nll ? ctx->u_zz.p : nullptr;
        L.fail = ctx->u_fail.p;
        CK(cudaEventRecord(ctx->ev[0], st), "event");
        CK(cudaMemcpyAsync(ctx->u_map.p, umap.data(), sizeof(int32_t) * C, cudaMemcpyHostToDevice, st), "copy");
        CK(cudaMemcpyAsync(ctx->u_sigma2.p, sig2.data(), sizeof(double) * C, cudaMemcpyHostToDevice, st), "copy");
        CK(cudaMemcpyAsync(ctx->own_mask.p, own.data(), (size_t)N, cudaMemcpyHostToDevice, st), "copy");
        CK(cudaMemsetAsync(ctx->u_loss.p, 0, sizeof(double) * N * U, st), "memset");
        CK(cudaMemsetAsync(ctx->u_fail.p, 0, (size_t)N * U, st), "memset");
        int r = run_cv(ctx, L);
        if (r) return r;
        launches = L.launches;
        // unique configs -> configs (and -2 log L per sigma2); zeros where this rank did
        // not evaluate, so a sum over ranks is exact
        CK(launch_expand(N, C, U, ctx->u_map.p, ctx->own_mask.p, ctx->train_off.p, ctx->u_sigma2.p, ctx->u_loss.p,
                         ctx->u_fail.p, L.logdet, L.zz, ctx->subset_loss.p, ctx->fail.p,
                         want_nll ? ctx->subset_nll.p : nullptr, st), "expand");
        ++launches;
        return PGPCV_OK;
    };
    if ((rc = join_ranks(ctx, local()))) return rc;

    // ---- combine (Alg.1 line 9) ----
    if (gather) {
        // each (s, c) entry has exactly one owner (others hold 0): the sums are exact, and
        // the global reductions below then run on identical arrays on every rank.
        if (want_cv && (rc = nccl_sum(ctx, ctx->subset_loss.p, (size_t)N * C, ncclFloat64))) return rc;
        if (want_nll && (rc = nccl_sum(ctx, ctx->subset_nll.p, (size_t)N * C, ncclFloat64))) return rc;
        if ((rc = nccl_sum(ctx, ctx->fail.p, (size_t)N * C, ncclUint8))) return rc;
    }
    double *d_loss = ctx->sums.p, *d_nll = ctx->sums.p + C;
    int32_t *d_st_loss = ctx->status.p, *d_st_nll = ctx->status.p + C;
    if (want_cv) {
        CK(launch_reduce(ctx->subset_loss.p, ctx->fail.p, ctx->val_off.p, N, C, d_loss, d_st_loss, st), "reduce");
        ++launches;
    }
    if (want_nll) {
        CK(launch_reduce(ctx->subset_nll.p, ctx->fail.p, nullptr, N, C, d_nll, d_st_nll, st), "reduce");
        ++launches;
    }
    if (multi && !gather) {
        // Alg.1 line 9 across GPUs: one all-reduce of the per-configuration [loss | nll]
        // vector, and a MIN all-reduce of the statuses.
        if (!want_cv) CK(cudaMemsetAsync(d_loss, 0, sizeof(double) * C, st), "memset");
        if (!want_nll) CK(cudaMemsetAsync(d_nll, 0, sizeof(double) * C, st), "memset");
        if (!want_cv) CK(cudaMemsetAsync(d_st_loss, 0xff, sizeof(int32_t) * C, st), "memset");
        if (!want_nll) CK(cudaMemsetAsync(d_st_nll, 0xff, sizeof(int32_t) * C, st), "memset");
        if ((rc = nccl_sum(ctx, ctx->sums.p, 2 * (size_t)C, ncclFloat64))) return rc;
        CK(launch_status_encode(ctx->status.p, 2 * C, -1, st), "status");
        if ((rc = nccl_sum(ctx, ctx->status.p, 2 * (size_t)C, ncclInt32, ncclMin))) return rc;
        CK(launch_status_encode(ctx->status.p, 2 * C, 0x7fffffff, st), "status");
        launches += 2;
    }
    std::vector<double> hsums(2 * (size_t)C);
    std::vector<int32_t> hstatus(2 * (size_t)C, -1);
    CK(cudaMemcpyAsync(hsums.data(), ctx->sums.p, sizeof(double) * 2 * C, cudaMemcpyDeviceToHost, st), "copy sums");
    CK(cudaMemcpyAsync(hstatus.data(), ctx->status.p, sizeof(int32_t) * 2 * C, cudaMemcpyDeviceToHost, st),
       "copy status");
    if (out->subset_loss)
        CK(cudaMemcpyAsync(out->subset_loss, ctx->subset_loss.p, sizeof(double) * N * C, cudaMemcpyDeviceToHost, st),
           "copy subset_loss");
    if (out->subset_nll)
        CK(cudaMemcpyAsync(out->subset_nll, ctx->subset_nll.p, sizeof(double) * N * C, cudaMemcpyDeviceToHost, st),
           "copy subset_nll");
    CK(cudaEventRecord(ctx->ev[3], st), "event");
    if ((rc = finish(ctx, "evaluate"))) return rc;
    ctx->cv_done = true;
    record_timing(ctx, L, launches, U);
    if (want_cv && (!multi || gather)) ctx->sel_C = C;  // every subset's loss is on this device

    bool any_fail = false;
    for (int c = 0; c < C; ++c) {
        const int32_t sl = want_cv ? hstatus[c] : -1, sn = want_nll ? hstatus[C + c] : -1;
        if (out->loss) out->loss[c] = hsums[c];
        if (out->nll) out->nll[c] = hsums[C + c];
        const int32_t f = first_fail(sl, sn);
        if (out->status) out->status[c] = f;
        any_fail |= f >= 0;
    }
    if (any_fail) return ctx->fail_with(PGPCV_ENUMERIC, "some configuration was not positive definite");
    return PGPCV_OK;
}

int pgpcv_cv_loss(pgpcv_ctx *ctx, const pgpcv_param *params, int32_t n_params, double *loss,
                  double *subset_loss, int32_t *status) {
    if (!ctx) return PGPCV_EINVAL;
    if (!loss) return ctx->fail_with(PGPCV_EINVAL, "NULL loss");
    pgpcv_outputs o{};
    o.loss = loss;
    o.subset_loss = subset_loss;
    o.status = status;
    return pgpcv_evaluate(ctx, params, n_params, &o);
}

int pgpcv_select(pgpcv_ctx *ctx, int32_t *best, double *rmspe, int32_t *local_best, double *local_rmspe,
                 int32_t *wins) {
    NvtxRange nvtx_("pgpcv_select");
    if (!ctx) return PGPCV_EINVAL;
    if (ctx->sel_C <= 0)
        return ctx->fail_with(PGPCV_ESTATE, "pgpcv_select needs a preceding CV evaluation whose per-subset "
                                            "losses are all on this device (world 1, or subset_loss requested)");
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    const int64_t N = ctx->N;
    const int32_t C = ctx->sel_C;
    CK(ctx->sel_rmspe.ensure(C), "alloc");
    CK(ctx->sel_local.ensure((size_t)N * C), "alloc");
    CK(ctx->sel_best.ensure(N + 1), "alloc");
    CK(ctx->sel_wins.ensure(C), "alloc");
    CK(launch_select(ctx->subset_loss.p, ctx->fail.p, ctx->val_off.p, ctx->sums.p, N, C, ctx->info.sum_m,
                     ctx->sel_rmspe.p, ctx->sel_local.p, ctx->sel_best.p, ctx->sel_wins.p, st), "select");
    if (best) CK(cudaMemcpyAsync(best, ctx->sel_best.p + N, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "copy");
    if (rmspe) CK(cudaMemcpyAsync(rmspe, ctx->sel_rmspe.p, sizeof(double) * C, cudaMemcpyDeviceToHost, st), "copy");
    if (local_best)
        CK(cudaMemcpyAsync(local_best, ctx->sel_best.p, sizeof(int32_t) * N, cudaMemcpyDeviceToHost, st), "copy");
    if (local_rmspe)
        CK(cudaMemcpyAsync(local_rmspe, ctx->sel_local.p, sizeof(double) * N * C, cudaMemcpyDeviceToHost, st),
           "copy");
    if (wins) CK(cudaMemcpyAsync(wins, ctx->sel_wins.p, sizeof(int32_t) * C, cudaMemcpyDeviceToHost, st), "copy");
    CK(cudaStreamSynchronize(st), "select");
    return PGPCV_OK;
}

int pgpcv_predict(pgpcv_ctx *ctx, const pgpcv_param *params, int32_t n_params, const int32_t *subset_config,
                  int32_t target_role, double *yhat, double *subset_sspe, double *sspe) {
    NvtxRange nvtx_("pgpcv_predict");
    if (!ctx) return PGPCV_EINVAL;
    if (!ctx->has_partition) return ctx->fail_with(PGPCV_ESTATE, "pgpcv_predict needs a partition");
    int rc = check_params(ctx, params, n_params);
    if (rc) return rc;
    if (target_role != PGPCV_ROLE_VALIDATION && target_role != PGPCV_ROLE_TEST)
        return ctx->fail_with(PGPCV_EINVAL, "target_role must be PGPCV_ROLE_VALIDATION or PGPCV_ROLE_TEST");
    const int64_t N = ctx->N;
    if (subset_config)
        for (int64_t s = 0; s < N; ++s)
            if (subset_config[s] < 0 || subset_config[s] >= n_params)
                return ctx->fail_with(PGPCV_EINVAL, "subset_config[%lld] = %d not in [0, %d)", (long long)s,
                                      subset_config[s], n_params);
    if ((rc = check_common(ctx))) return rc;
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    const bool test = target_role == PGPCV_ROLE_TEST;
    const std::vector<int64_t> &hoff = test ? ctx->h_test_off : ctx->h_val_off;
    const int64_t n_tgt = hoff[N];

    CvLaunch L;
    L.flags = kCvPredict;
    L.params = params;
    L.C = n_params;
    L.out_C = 1;
    L.tgt_off = test ? ctx->test_off.p : ctx->val_off.p;
    L.h_tgt_off = hoff.data();
    L.gx = test ? ctx->gx.p : ctx->vx.p;
    L.gy = test ? ctx->gy.p : ctx->vy.p;
    L.gv = test ? ctx->gv.p : ctx->vv.p;
    std::vector<uint8_t> work(N);
    for (int64_t s = 0; s < N; ++s) work[s] = hoff[s + 1] > hoff[s];
    assign_owned(ctx, work);
    for (int64_t s = 0; s < N; ++s) {
        const int64_t k = ctx->h_train_off[s + 1] - ctx->h_train_off[s];
        const int64_t m = hoff[s + 1] - hoff[s];
        if (!ctx->owned[s] || m == 0) continue;
        L.items.push_back(make_int2((int)s, subset_config ? subset_config[s] : 0));
        const double kd = (double)k, md = (double)m;
        L.flops += kd * kd * kd / 3.0 + kd * kd / 2.0 + kd / 6.0 + 2.0 * kd * kd + 2.0 * md * kd + 3.0 * md;
    }
    int launches = 0;
    auto local = [&]() -> int {
        CK(ctx->p_sub.ensure(N), "alloc");
        CK(ctx->p_fail.ensure(N), "alloc");
        CK(ctx->p_yhat.ensure(std::max<int64_t>(n_tgt, 1)), "alloc");
        CK(ctx->p_sum.ensure(1), "alloc");
        CK(ctx->p_status.ensure(1), "alloc");
        L.subset_loss = ctx->p_sub.p;
        L.fail = ctx->p_fail.p;
        L.yhat = yhat ? ctx->p_yhat.p : nullptr;
        CK(cudaEventRecord(ctx->ev[0], st), "event");
        CK(cudaMemsetAsync(ctx->p_sub.p, 0, sizeof(double) * N, st), "memset");
        CK(cudaMemsetAsync(ctx->p_fail.p, 0, (size_t)N, st), "memset");
        if (yhat) CK(cudaMemsetAsync(ctx->p_yhat.p, 0, sizeof(double) * std::max<int64_t>(n_tgt, 1), st), "memset");
        int r = run_cv(ctx, L);
        launches = L.launches;
        return r;
    };
    if ((rc = join_ranks(ctx, local()))) return rc;
    if (ctx->world > 1) {  // exclusive owners: exact sums
        if ((rc = nccl_sum(ctx, ctx->p_sub.p, (size_t)N, ncclFloat64))) return rc;
        if ((rc = nccl_sum(ctx, ctx->p_fail.p, (size_t)N, ncclUint8))) return rc;
        if (yhat && n_tgt && (rc = nccl_sum(ctx, ctx->p_yhat.p, (size_t)n_tgt, ncclFloat64))) return rc;
    }
    CK(launch_reduce(ctx->p_sub.p, ctx->p_fail.p, L.tgt_off, N, 1, ctx->p_sum.p, ctx->p_status.p, st), "reduce");
    ++launches;
    double total = 0;
    int32_t status = -1;
    CK(cudaMemcpyAsync(&total, ctx->p_sum.p, sizeof(double), cudaMemcpyDeviceToHost, st), "copy");
    CK(cudaMemcpyAsync(&status, ctx->p_status.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "copy");
    if (subset_sspe) CK(cudaMemcpyAsync(subset_sspe, ctx->p_sub.p, sizeof(double) * N, cudaMemcpyDeviceToHost, st), "copy");
    if (yhat && n_tgt)
        CK(cudaMemcpyAsync(yhat, ctx->p_yhat.p, sizeof(double) * n_tgt, cudaMemcpyDeviceToHost, st), "copy");
    CK(cudaEventRecord(ctx->ev[3], st), "event");
    if ((rc = finish(ctx, "predict"))) return rc;
    ctx->cv_done = true;
    record_timing(ctx, L, launches, n_params);
    if (sspe) *sspe = total;
    if (status >= 0) return ctx->fail_with(PGPCV_ENUMERIC, "subset %d was not positive definite", status);
    return PGPCV_OK;
}

int pgpcv_gls(pgpcv_ctx *ctx, const double *X, int32_t p, pgpcv_param param, double *beta, double *xtmx,
              double *xtmy) {
    NvtxRange nvtx_("pgpcv_gls");
    if (!ctx) return PGPCV_EINVAL;
    if (!ctx->has_partition) return ctx->fail_with(PGPCV_ESTATE, "pgpcv_gls needs a partition");
    if (p < 1 || p > kMaxCovariates) return ctx->fail_with(PGPCV_EINVAL, "need 1 <= p <= %d covariates", kMaxCovariates);
    if (!X || !beta) return ctx->fail_with(PGPCV_EINVAL, "NULL X or beta");
    int rc = check_params(ctx, &param, 1);
    if (rc) return rc;
    if ((rc = check_common(ctx))) return rc;
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    const int64_t N = ctx->N, n = ctx->n, sum_k = ctx->info.sum_k;
    const int W = (p + 1) * p;
    CvLaunch L;
    L.flags = kCvGls;
    L.params = &param;
    L.C = 1;
    L.out_C = 1;
    L.tgt_off = ctx->val_off.p;
    L.h_tgt_off = ctx->h_val_off.data();
    L.gx = ctx->vx.p;
    L.gy = ctx->vy.p;
    L.gv = ctx->vv.p;
    L.p = p;
    std::vector<uint8_t> work(N);
    for (int64_t s = 0; s < N; ++s) work[s] = ctx->h_train_off[s + 1] > ctx->h_train_off[s];
    assign_owned(ctx, work);
    for (int64_t s = 0; s < N; ++s) {
        const int64_t k = ctx->h_train_off[s + 1] - ctx->h_train_off[s];
        if (!ctx->owned[s] || k == 0) continue;
        L.items.push_back(make_int2((int)s, 0));
        const double kd = (double)k;
        // Cholesky + (p+1) forward (bordered) and backward solves + core-row sums
        L.flops += kd * kd * kd / 3.0 + kd * kd / 2.0 + kd / 6.0 + (p + 1) * (2.0 * kd * kd + 2.0 * kd * p);
    }
    int launches = 0;
    auto local = [&]() -> int {
        CK(ctx->g_X.ensure((size_t)n * p), "alloc");
        CK(ctx->g_tX.ensure((size_t)sum_k * p), "alloc");
        CK(ctx->g_part.ensure((size_t)N * W), "alloc");
        CK(ctx->g_sums.ensure(W), "alloc");
        CK(ctx->g_beta.ensure(p), "alloc");
        CK(ctx->p_fail.ensure(N), "alloc");
        CK(ctx->p_status.ensure(1), "alloc");
        L.fail = ctx->p_fail.p;
        L.tX = ctx->g_tX.p;
        L.gls_out = ctx->g_part.p;
        CK(cudaEventRecord(ctx->ev[0], st), "event");
        CK(cudaMemcpyAsync(ctx->g_X.p, X, sizeof(double) * n * p, cudaMemcpyHostToDevice, st), "copy X");
        CK(launch_gather_rows(sum_k, ctx->train_idx.p, ctx->g_X.p, p, ctx->g_tX.p, st), "gather X");
        CK(cudaMemsetAsync(ctx->g_part.p, 0, sizeof(double) * N * W, st), "memset");
        CK(cudaMemsetAsync(ctx->p_fail.p, 0, (size_t)N, st), "memset");
        int r = run_cv(ctx, L);
        launches = 1 + L.launches;
        return r;
    };
    if ((rc = join_ranks(ctx, local()))) return rc;
    if (ctx->world > 1) {  // exclusive owners: exact sums
        if ((rc = nccl_sum(ctx, ctx->g_part.p, (size_t)N * W, ncclFloat64))) return rc;
        if ((rc = nccl_sum(ctx, ctx->p_fail.p, (size_t)N, ncclUint8))) return rc;
    }
    CK(launch_gls_solve(ctx->g_part.p, ctx->p_fail.p, N, p, ctx->g_sums.p, ctx->g_beta.p, ctx->p_status.p, st),
       "gls solve");
    ++launches;
    std::vector<double> sums(W);
    int32_t status = 0;
    CK(cudaMemcpyAsync(beta, ctx->g_beta.p, sizeof(double) * p, cudaMemcpyDeviceToHost, st), "copy");
    CK(cudaMemcpyAsync(sums.data(), ctx->g_sums.p, sizeof(double) * W, cudaMemcpyDeviceToHost, st), "copy");
    CK(cudaMemcpyAsync(&status, ctx->p_status.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "copy");
    CK(cudaEventRecord(ctx->ev[3], st), "event");
    if ((rc = finish(ctx, "gls"))) return rc;
    ctx->cv_done = true;
    record_timing(ctx, L, launches, 1);
    if (xtmx) memcpy(xtmx, sums.data(), sizeof(double) * p * p);
    if (xtmy) memcpy(xtmy, sums.data() + p * p, sizeof(double) * p);
    if (std::isnan(sums[0])) return ctx->fail_with(PGPCV_ENUMERIC, "a subset was not positive definite");
    if (status) return ctx->fail_with(PGPCV_ENUMERIC, "X^T M^-1 X is singular");
    return PGPCV_OK;
}

int pgpcv_partition_export_test(pgpcv_ctx *ctx, int64_t *test_off, int32_t *test_idx) {
    if (!ctx) return PGPCV_EINVAL;
    if (!ctx->has_partition) return ctx->fail_with(PGPCV_ESTATE, "no partition");
    cudaSetDevice(ctx->device);
    const int64_t N = ctx->N;
    if (test_off) memcpy(test_off, ctx->h_test_off.data(), sizeof(int64_t) * (N + 1));
    if (test_idx && ctx->info.n_test)
        CK(cudaMemcpyAsync(test_idx, ctx->test_idx.p, sizeof(int32_t) * ctx->info.n_test, cudaMemcpyDeviceToHost,
                           ctx->stream), "copy test_idx");
    CK(cudaStreamSynchronize(ctx->stream), "export");
    return PGPCV_OK;
}

int pgpcv_device_math(pgpcv_ctx *ctx, int32_t fn, int64_t n, const double *x, double *y) {
    if (!ctx) return PGPCV_EINVAL;
    if (fn < PGPCV_MATH_EXP_NEG || fn > PGPCV_MATH_RSQRT || n < 0 || (n > 0 && (!x || !y)))
        return ctx->fail_with(PGPCV_EINVAL, "bad function id, n or NULL array");
    if (n == 0) return PGPCV_OK;
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    DevBuf<double> dx, dy;
    CK(dx.ensure(n), "alloc");
    CK(dy.ensure(n), "alloc");
    CK(cudaMemcpyAsync(dx.p, x, sizeof(double) * n, cudaMemcpyHostToDevice, st), "copy");
    CK(launch_device_math(fn, n, dx.p, dy.p, st), "device math");
    CK(cudaMemcpyAsync(y, dy.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st), "copy");
    CK(cudaStreamSynchronize(st), "device math");
    return PGPCV_OK;
}

int pgpcv_last_timing(const pgpcv_ctx *ctx, pgpcv_timing *out) {
    if (!ctx || !out) return PGPCV_EINVAL;
    if (!ctx->has_timing) return PGPCV_ESTATE;
    *out = ctx->timing;
    return PGPCV_OK;
}

int pgpcv_lpt_assign(int64_t n_items, const double *cost, int32_t world, int32_t *owner) {
    if (n_items < 0 || world < 1 || (n_items > 0 && (!cost || !owner))) return PGPCV_EINVAL;
    std::vector<int64_t> order(n_items);
    for (int64_t i = 0; i < n_items; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return cost[a] > cost[b]; });
    std::vector<double> load(world, 0.0);
    for (int64_t i : order) {
        int best = 0;
        for (int r = 1; r < world; ++r)
            if (load[r] < load[best]) best = r;
        owner[i] = best;
        load[best] += cost[i];
    }
    return PGPCV_OK;
}

}  // extern "C"
