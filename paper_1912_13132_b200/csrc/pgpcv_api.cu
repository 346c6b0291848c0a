// pgpcv_api.cu -- the C ABI of libpgpcv (include/pgpcv.h): argument checking, device
// memory and stream ownership, work scheduling (LPT), the NCCL combine step, timing.
// Every numerical step runs in the kernels of partition.cu and cv_kernel.cu.
#include <dlfcn.h>

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
#include "pgpcv_internal.h"

using namespace pgpcv;

namespace {

// ------------------------------------------------------------------ device buffers
template <typename T>
struct DevBuf {
    T *p = nullptr;
    size_t cap = 0;  // elements
    ~DevBuf() { release(); }
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
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                              ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char *(*getErrorString)(ncclResult_t) = nullptr;
};

NcclApi &nccl() {
    static NcclApi api;
    static bool tried = false;
    if (tried) return api;
    tried = true;
    // Prefer an already-loaded libnccl (torch's bundled copy) so one process never holds two.
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) {
        const char *env = getenv("PGPCV_NCCL_LIB");
        if (env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        api.why = std::string("cannot dlopen libnccl.so.2: ") + dlerror();
        return api;
    }
    api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
    api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
    api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
    api.getErrorString = (decltype(api.getErrorString))dlsym(h, "ncclGetErrorString");
    api.ok = api.getUniqueId && api.commInitRank && api.allReduce && api.commDestroy &&
             api.getErrorString;
    if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
    return api;
}

std::string g_create_error;

// status: -1 -> INT32_MAX so a MIN all-reduce yields the smallest failing subset, and back
__global__ void status_encode(int32_t *st, int32_t C, int32_t sentinel) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < C && st[c] == sentinel) st[c] = (sentinel == -1) ? 0x7fffffff : -1;
}

double subset_flops(double k, double m) {
    // Cholesky k^3/3 + k^2/2 + k/6, two triangular solves 2k^2,
    // prediction 2mk, residual and square 3m.  exp/sqrt are not counted.
    return k * k * k / 3.0 + k * k / 2.0 + k / 6.0 + 2.0 * k * k + 2.0 * m * k + 3.0 * m;
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
    std::string err;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};

    // partition state
    bool has_partition = false;
    int64_t n = 0, N = 0;
    int32_t kx = 0, ky = 0;
    DevBuf<double> px, py, pv;
    DevBuf<uint8_t> prole;
    DevBuf<double> bounds;  // ex, lox, hix, ey, loy, hiy
    DevBuf<unsigned int> cnt, cur;
    DevBuf<unsigned long long> stats;
    DevBuf<int64_t> train_off, val_off;
    DevBuf<int32_t> train_idx, val_idx;
    DevBuf<uint32_t> bitmap;
    DevBuf<double> tx, ty, tv, vx, vy, vv;
    std::vector<int64_t> h_train_off, h_val_off;
    pgpcv_partition_info info{};

    // sharding
    int rank = 0, world = 1;
    ncclComm_t comm = nullptr;
    bool cv_done = false;
    std::vector<uint8_t> owned;

    // cv_loss buffers
    DevBuf<double> work;
    DevBuf<double> params;
    DevBuf<int2> items;
    DevBuf<unsigned int> counter;
    DevBuf<double> subset_loss, loss;
    DevBuf<uint8_t> fail;
    DevBuf<int32_t> status;
    int blocks_per_sm = 0;
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

void assign_owned(pgpcv_ctx *ctx) {
    ctx->owned.assign(ctx->N, 1);
    if (ctx->world <= 1) return;
    std::vector<double> cost(ctx->N);
    for (int64_t s = 0; s < ctx->N; ++s) {
        const double k = (double)(ctx->h_train_off[s + 1] - ctx->h_train_off[s]);
        const double m = (double)(ctx->h_val_off[s + 1] - ctx->h_val_off[s]);
        cost[s] = m > 0 ? k * k * k : 0.0;  // the rule documented in pgpcv.h
    }
    std::vector<int32_t> owner(ctx->N);
    pgpcv_lpt_assign(ctx->N, cost.data(), ctx->world, owner.data());
    for (int64_t s = 0; s < ctx->N; ++s) ctx->owned[s] = owner[s] == ctx->rank;
}

int partition_impl(pgpcv_ctx *ctx, int64_t n, const double *x, const double *y, const double *v,
                   const uint8_t *role, pgpcv_rect d, int32_t kx, int32_t ky, double delta,
                   pgpcv_partition_info *info_out) {
    cudaStream_t st = ctx->stream;
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
    Axis ax{b, b + (kx + 1), b + (kx + 1) + kx, kx};
    double *b2 = b + (kx + 1) + 2 * kx;
    Axis ay{b2, b2 + (ky + 1), b2 + (ky + 1) + ky, ky};

    const int64_t N = (int64_t)kx * ky;
    ctx->N = N;
    ctx->n = n;
    ctx->kx = kx;
    ctx->ky = ky;
    // K1 count, K2 scan
    CK(ctx->cnt.ensure(2 * N), "alloc counts");
    CK(ctx->cur.ensure(2 * N), "alloc cursors");
    CK(ctx->train_off.ensure(N + 1), "alloc offsets");
    CK(ctx->val_off.ensure(N + 1), "alloc offsets");
    CK(cudaMemsetAsync(ctx->cnt.p, 0, sizeof(unsigned) * 2 * N, st), "memset");
    CK(launch_count(n, x, y, role, ax, ay, ctx->cnt.p, ctx->cnt.p + N, st), "count kernel");
    CK(launch_scan(ctx->cnt.p, N, ctx->train_off.p, st), "scan kernel");
    CK(launch_scan(ctx->cnt.p + N, N, ctx->val_off.p, st), "scan kernel");
    ctx->h_train_off.resize(N + 1);
    ctx->h_val_off.resize(N + 1);
    CK(cudaMemcpyAsync(ctx->h_train_off.data(), ctx->train_off.p, sizeof(int64_t) * (N + 1),
                       cudaMemcpyDeviceToHost, st), "copy offsets");
    CK(cudaMemcpyAsync(ctx->h_val_off.data(), ctx->val_off.p, sizeof(int64_t) * (N + 1),
                       cudaMemcpyDeviceToHost, st), "copy offsets");
    CK(cudaStreamSynchronize(st), "scan");
    const int64_t sum_k = ctx->h_train_off[N], sum_m = ctx->h_val_off[N];
    if (sum_k >= (int64_t)1 << 31 || sum_m >= (int64_t)1 << 31)
        return ctx->fail_with(PGPCV_EINVAL, "more than 2^31 memberships");
    // K3 scatter + per-segment sort into ascending index order
    CK(ctx->train_idx.ensure(sum_k), "alloc train_idx");
    CK(ctx->val_idx.ensure(sum_m), "alloc val_idx");
    CK(cudaMemsetAsync(ctx->cur.p, 0, sizeof(unsigned) * 2 * N, st), "memset");
    CK(launch_scatter(n, x, y, role, ax, ay, ctx->train_off.p, ctx->val_off.p, ctx->cur.p,
                      ctx->cur.p + N, ctx->train_idx.p, ctx->val_idx.p, st), "scatter kernel");
    int64_t max_k = 0, max_m = 0, empty = 0;
    for (int64_t s = 0; s < N; ++s) {
        max_k = std::max(max_k, ctx->h_train_off[s + 1] - ctx->h_train_off[s]);
        const int64_t m = ctx->h_val_off[s + 1] - ctx->h_val_off[s];
        max_m = std::max(max_m, m);
        empty += m == 0;
    }
    CK(launch_segsort_small(ctx->train_idx.p, ctx->train_off.p, N, max_k, st), "segsort");
    CK(launch_segsort_small(ctx->val_idx.p, ctx->val_off.p, N, max_m, st), "segsort");
    for (int which = 0; which < 2; ++which) {
        const std::vector<int64_t> &off = which ? ctx->h_val_off : ctx->h_train_off;
        int32_t *idx = which ? ctx->val_idx.p : ctx->train_idx.p;
        for (int64_t s = 0; s < N; ++s) {
            const int64_t len = off[s + 1] - off[s];
            if (len > kSmallSortMax) {
                CK(ctx->bitmap.ensure((n + 31) / 32), "alloc bitmap");
                CK(sort_long_segment(idx, off[s], len, n, ctx->bitmap.p, st), "long sort");
            }
        }
    }
    // K4 staging gather (subset-contiguous SoA)
    CK(ctx->tx.ensure(sum_k), "alloc");
    CK(ctx->ty.ensure(sum_k), "alloc");
    CK(ctx->tv.ensure(sum_k), "alloc");
    CK(ctx->vx.ensure(sum_m), "alloc");
    CK(ctx->vy.ensure(sum_m), "alloc");
    CK(ctx->vv.ensure(sum_m), "alloc");
    CK(launch_gather(sum_k, ctx->train_idx.p, x, y, v, ctx->tx.p, ctx->ty.p, ctx->tv.p, st), "gather");
    CK(launch_gather(sum_m, ctx->val_idx.p, x, y, v, ctx->vx.p, ctx->vy.p, ctx->vv.p, st), "gather");
    CK(cudaStreamSynchronize(st), "partition");

    pgpcv_partition_info &info = ctx->info;
    info.n_subsets = N;
    info.sum_k = sum_k;
    info.sum_m = sum_m;
    info.max_k = max_k;
    info.max_m = max_m;
    info.n_empty_val = empty;
    info.n_train = (int64_t)hstats[1];
    info.n_val = (int64_t)hstats[2];
    ctx->has_partition = true;
    ctx->cv_done = false;
    assign_owned(ctx);
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
    for (auto &ev : ctx->ev) cudaEventCreate(&ev);
    if ((e = cv_kernel_occupancy(&ctx->blocks_per_sm)) != cudaSuccess || ctx->blocks_per_sm < 1) {
        g_create_error = std::string("cv kernel cannot be resident: ") + cudaGetErrorString(e);
        pgpcv_destroy(ctx);
        return PGPCV_ECUDA;
    }
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
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
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
    return partition_impl(ctx, n, ctx->px.p, ctx->py.p, ctx->pv.p, ctx->prole.p, domain, kx, ky,
                          delta, info_out);
}

int pgpcv_partition_device(pgpcv_ctx *ctx, int64_t n, const double *d_x, const double *d_y,
                           const double *d_value, const uint8_t *d_role, pgpcv_rect domain,
                           int32_t kx, int32_t ky, double delta, pgpcv_partition_info *info_out) {
    if (!ctx) return PGPCV_EINVAL;
    int rc = check_partition_args(ctx, n, d_x, d_y, d_value, d_role, domain, kx, ky, delta);
    if (rc) return rc;
    cudaSetDevice(ctx->device);
    return partition_impl(ctx, n, d_x, d_y, d_value, d_role, domain, kx, ky, delta, info_out);
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
    if (!ctx) return PGPCV_EINVAL;
    if (world < 1 || rank < 0 || rank >= world)
        return ctx->fail_with(PGPCV_EINVAL, "need 0 <= rank < world");
    if (!ctx->has_partition) return ctx->fail_with(PGPCV_ESTATE, "pgpcv_shard needs a partition");
    if (ctx->cv_done)
        return ctx->fail_with(PGPCV_ESTATE, "pgpcv_shard after pgpcv_cv_loss on this partition");
    cudaSetDevice(ctx->device);
    if (ctx->comm) {
        nccl().commDestroy(ctx->comm);
        ctx->comm = nullptr;
    }
    ctx->rank = rank;
    ctx->world = world;
    if (world > 1) {
        if (!nccl_unique_id) return ctx->fail_with(PGPCV_EINVAL, "world > 1 needs an ncclUniqueId");
        NcclApi &api = nccl();
        if (!api.ok) return ctx->fail_with(PGPCV_ENCCL, "%s", api.why.c_str());
        ncclUniqueId id;
        memcpy(&id, nccl_unique_id, sizeof id);
        ncclResult_t r = api.commInitRank(&ctx->comm, world, id, rank);
        if (r != ncclSuccess) {
            ctx->comm = nullptr;
            ctx->world = 1;
            ctx->rank = 0;
            return ctx->fail_with(PGPCV_ENCCL, "ncclCommInitRank: %s", api.getErrorString(r));
        }
    }
    assign_owned(ctx);
    return PGPCV_OK;
}

int pgpcv_cv_loss(pgpcv_ctx *ctx, const pgpcv_param *params, int32_t n_params, double *loss,
                  double *subset_loss, int32_t *status) {
    if (!ctx) return PGPCV_EINVAL;
    if (!ctx->has_partition) return ctx->fail_with(PGPCV_ESTATE, "pgpcv_cv_loss needs a partition");
    if (n_params < 1 || !params || !loss) return ctx->fail_with(PGPCV_EINVAL, "bad params/loss");
    for (int c = 0; c < n_params; ++c) {
        const pgpcv_param &p = params[c];
        if (!(p.range > 0) || !(p.sigma2 > 0) || !(p.nugget >= 0) || !std::isfinite(p.range) ||
            !std::isfinite(p.sigma2) || !std::isfinite(p.nugget))
            return ctx->fail_with(PGPCV_EINVAL, "config %d: need range > 0, sigma2 > 0, nugget >= 0", c);
    }
    if (ctx->info.sum_m == 0) return ctx->fail_with(PGPCV_EEMPTY, "no subset has validation data");
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    const int64_t N = ctx->N;
    const int32_t C = n_params;

    // work items: owned subsets with validation data, descending k (LPT), all configs
    std::vector<int32_t> subs;
    for (int64_t s = 0; s < N; ++s)
        if (ctx->owned[s] && ctx->h_val_off[s + 1] > ctx->h_val_off[s]) subs.push_back((int32_t)s);
    std::stable_sort(subs.begin(), subs.end(), [&](int32_t a, int32_t b) {
        return ctx->h_train_off[a + 1] - ctx->h_train_off[a] > ctx->h_train_off[b + 1] - ctx->h_train_off[b];
    });
    int64_t kmax = 0;
    double flops = 0;
    std::vector<int2> items;
    items.reserve(subs.size() * C);
    for (int32_t s : subs) {
        const int64_t k = ctx->h_train_off[s + 1] - ctx->h_train_off[s];
        const int64_t m = ctx->h_val_off[s + 1] - ctx->h_val_off[s];
        kmax = std::max(kmax, k);
        for (int32_t c = 0; c < C; ++c) items.push_back(make_int2(s, c));
        flops += C * subset_flops((double)k, (double)m);
    }
    if (kmax > cv_kernel_max_k())
        return ctx->fail_with(PGPCV_EINVAL, "a subset has %lld training points (max %d)",
                              (long long)kmax, cv_kernel_max_k());
    const int64_t n_items = (int64_t)items.size();
    if (n_items >= ((int64_t)1 << 31)) return ctx->fail_with(PGPCV_EINVAL, "too many work items");

    std::vector<double> hp(3 * (size_t)C);
    for (int c = 0; c < C; ++c) {
        hp[3 * c] = params[c].range;
        hp[3 * c + 1] = params[c].sigma2;
        hp[3 * c + 2] = params[c].nugget;
    }
    CK(ctx->params.ensure(3 * (size_t)C), "alloc params");
    CK(ctx->items.ensure(std::max<int64_t>(n_items, 1)), "alloc items");
    CK(ctx->counter.ensure(1), "alloc counter");
    CK(ctx->subset_loss.ensure((size_t)N * C), "alloc subset_loss");
    CK(ctx->fail.ensure((size_t)N * C), "alloc fail");
    CK(ctx->loss.ensure(C), "alloc loss");
    CK(ctx->status.ensure(C), "alloc status");

    // factor workspace: one column-major (k+1) x k factor per resident CTA
    int slots = (int)std::min<int64_t>((int64_t)ctx->sms * ctx->blocks_per_sm, std::max<int64_t>(n_items, 1));
    if (const char *env = getenv("PGPCV_MAX_SLOTS")) {  // diagnostics: cap resident CTAs
        const int cap = atoi(env);
        if (cap > 0) slots = std::min(slots, cap);
    }
    const size_t slot_stride = cv_kernel_slot_doubles(kmax);
    while (true) {
        cudaError_t e = ctx->work.ensure((size_t)slots * slot_stride);
        if (e == cudaSuccess) break;
        if (slots == 1) return ctx->cuda_fail(e, "alloc factor workspace");
        slots = std::max(1, slots / 2);
    }

    CK(cudaEventRecord(ctx->ev[0], st), "event");
    CK(cudaMemcpyAsync(ctx->params.p, hp.data(), sizeof(double) * hp.size(), cudaMemcpyHostToDevice, st),
       "copy params");
    if (n_items)
        CK(cudaMemcpyAsync(ctx->items.p, items.data(), sizeof(int2) * n_items, cudaMemcpyHostToDevice, st),
           "copy items");
    CK(cudaMemsetAsync(ctx->counter.p, 0, sizeof(unsigned), st), "memset");
    CK(cudaMemsetAsync(ctx->subset_loss.p, 0, sizeof(double) * N * C, st), "memset");
    CK(cudaMemsetAsync(ctx->fail.p, 0, (size_t)N * C, st), "memset");
    int launches = 0;
    CK(cudaEventRecord(ctx->ev[1], st), "event");
    if (n_items) {
        CvArgs a;
        a.train_off = ctx->train_off.p;
        a.val_off = ctx->val_off.p;
        a.tx = ctx->tx.p;
        a.ty = ctx->ty.p;
        a.tv = ctx->tv.p;
        a.vx = ctx->vx.p;
        a.vy = ctx->vy.p;
        a.vv = ctx->vv.p;
        a.params = ctx->params.p;
        a.C = C;
        a.items = ctx->items.p;
        a.n_items = (int32_t)n_items;
        a.counter = ctx->counter.p;
        a.work = ctx->work.p;
        a.slot_stride = slot_stride;
        a.subset_loss = ctx->subset_loss.p;
        a.fail = ctx->fail.p;
        CK(launch_cv_kernel(a, slots, st), "cv kernel launch");
        ++launches;
    }
    CK(cudaEventRecord(ctx->ev[2], st), "event");

    NcclApi &api = nccl();
    const bool multi = ctx->world > 1;
    if (multi && subset_loss) {
        // each (s, c) entry has exactly one owner (others hold 0): the sum is exact, and the
        // global reduction below then runs on identical arrays on every rank.
        ncclResult_t r = api.allReduce(ctx->subset_loss.p, ctx->subset_loss.p, (size_t)N * C,
                                       ncclFloat64, ncclSum, ctx->comm, st);
        if (r == ncclSuccess)
            r = api.allReduce(ctx->fail.p, ctx->fail.p, (size_t)N * C, ncclUint8, ncclSum, ctx->comm, st);
        if (r != ncclSuccess) return ctx->fail_with(PGPCV_ENCCL, "ncclAllReduce: %s", api.getErrorString(r));
    }
    CK(launch_reduce(ctx->subset_loss.p, ctx->fail.p, N, C, ctx->loss.p, ctx->status.p, st), "reduce");
    ++launches;
    if (multi && !subset_loss) {
        // Alg.1 line 9 across GPUs: one all-reduce of the per-configuration loss vector.
        ncclResult_t r = api.allReduce(ctx->loss.p, ctx->loss.p, C, ncclFloat64, ncclSum, ctx->comm, st);
        status_encode<<<(C + 127) / 128, 128, 0, st>>>(ctx->status.p, C, -1);
        ++launches;
        if (r == ncclSuccess)
            r = api.allReduce(ctx->status.p, ctx->status.p, C, ncclInt32, ncclMin, ctx->comm, st);
        status_encode<<<(C + 127) / 128, 128, 0, st>>>(ctx->status.p, C, 0x7fffffff);
        ++launches;
        if (r != ncclSuccess) return ctx->fail_with(PGPCV_ENCCL, "ncclAllReduce: %s", api.getErrorString(r));
    }
    std::vector<int32_t> hstatus(C);
    CK(cudaMemcpyAsync(loss, ctx->loss.p, sizeof(double) * C, cudaMemcpyDeviceToHost, st), "copy loss");
    CK(cudaMemcpyAsync(hstatus.data(), ctx->status.p, sizeof(int32_t) * C, cudaMemcpyDeviceToHost, st),
       "copy status");
    if (subset_loss)
        CK(cudaMemcpyAsync(subset_loss, ctx->subset_loss.p, sizeof(double) * N * C, cudaMemcpyDeviceToHost, st),
           "copy subset_loss");
    CK(cudaEventRecord(ctx->ev[3], st), "event");
    CK(cudaStreamSynchronize(st), "cv_loss");
    CK(cudaGetLastError(), "cv_loss");
    ctx->cv_done = true;

    float kms = 0, tms = 0;
    cudaEventElapsedTime(&kms, ctx->ev[1], ctx->ev[2]);
    cudaEventElapsedTime(&tms, ctx->ev[0], ctx->ev[3]);
    ctx->timing.kernel_ms = kms;
    ctx->timing.total_ms = tms;
    ctx->timing.flops = flops;
    ctx->timing.n_evals = n_items;
    ctx->timing.launches = launches;
    ctx->timing.n_slots = slots;
    ctx->has_timing = true;

    bool any_fail = false;
    for (int c = 0; c < C; ++c) {
        if (status) status[c] = hstatus[c];
        any_fail |= hstatus[c] >= 0;
    }
    if (any_fail) return ctx->fail_with(PGPCV_ENUMERIC, "some configuration was not positive definite");
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
