/* loopback_nccl.c -- TEST INFRASTRUCTURE ONLY (never linked into libpgpcv, never used by the
 * product path): a stand-in for the eight NCCL entry points libpgpcv binds, whose all-reduce
 * runs between the processes of one host through a POSIX shared-memory segment.
 *
 * Why: NCCL refuses two ranks on one GPU, and every GPU box of this build has one GPU, so the
 * library's world > 1 path (pgpcv_shard, LPT ownership, the gather / vector combines, the
 * status MIN all-reduce, the error-flag lockstep) could not run on hardware with real NCCL.
 * With PGPCV_NCCL_LIB pointing at this shim, two processes share cuda:0 and run exactly that
 * library code; only the transport differs (host memory instead of NVLink).
 *
 * Semantics: every call is synchronous on the host -- the stream is synchronised, the send
 * buffer copied to this rank's slot, a process barrier, the reduction over the slots in rank
 * order (identical bits on every rank), a second barrier, the result copied to recv.  Device
 * copies go through the driver API (shared by every CUDA runtime instance in the process),
 * on the caller's stream, each followed by a stream synchronisation.
 * Build: gcc -O2 -shared -fPIC -I<nccl include> loopback_nccl.c -o libloopback_nccl.so -ldl -lrt
 */
#define _GNU_SOURCE
#include <dlfcn.h>
#include <fcntl.h>
#include <sched.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#include <nccl.h>

#define SLOT_BYTES (8u << 20)

typedef struct {
    int nranks;
    int count; /* barrier arrivals */
    int gen;   /* barrier generation */
    char pad[52];
} Hdr;

struct ncclComm {
    Hdr *seg;
    size_t seg_bytes;
    int rank, nranks;
    char name[128];
    long seq; /* all-reduces issued (trace) */
    char *tmp;
};

typedef int (*sync_fn)(void *);
typedef int (*d2h_fn)(void *, unsigned long long, size_t, void *);
typedef int (*h2d_fn)(unsigned long long, const void *, size_t, void *);
static sync_fn p_sync;
static d2h_fn p_d2h;
static h2d_fn p_h2d;

static int bind_driver(void) {
    if (p_sync) return 0;
    void *h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return -1;
    p_sync = (sync_fn)dlsym(h, "cuStreamSynchronize");
    /* copies on the caller's stream, then a stream sync: a synchronous cuMemcpyHtoD from
     * pageable memory may return before its DMA lands and is not ordered with the caller's
     * non-blocking stream (a later read on that stream could see the old value) */
    p_d2h = (d2h_fn)dlsym(h, "cuMemcpyDtoHAsync_v2");
    p_h2d = (h2d_fn)dlsym(h, "cuMemcpyHtoDAsync_v2");
    return (p_sync && p_d2h && p_h2d) ? 0 : -1;
}

static void barrier(Hdr *s) {
    const int g = __atomic_load_n(&s->gen, __ATOMIC_ACQUIRE);
    if (__atomic_add_fetch(&s->count, 1, __ATOMIC_ACQ_REL) == s->nranks) {
        __atomic_store_n(&s->count, 0, __ATOMIC_RELAXED);
        __atomic_add_fetch(&s->gen, 1, __ATOMIC_RELEASE);
    } else {
        while (__atomic_load_n(&s->gen, __ATOMIC_ACQUIRE) == g) sched_yield();
    }
}

static char *slot(ncclComm_t c, int r) { return (char *)c->seg + sizeof(Hdr) + (size_t)r * SLOT_BYTES; }

ncclResult_t ncclGetVersion(int *v) { *v = 0; return ncclSuccess; }
const char *ncclGetErrorString(ncclResult_t r) { return r == ncclSuccess ? "success (loopback)" : "loopback error"; }

ncclResult_t ncclGetUniqueId(ncclUniqueId *id) {
    struct timespec ts;
    clock_gettime(CLOCK_REALTIME, &ts);
    memset(id, 0, sizeof *id);
    snprintf(id->internal, sizeof id->internal, "/pgpcv_loopback_%d_%lld", (int)getpid(),
             (long long)ts.tv_sec * 1000000000LL + ts.tv_nsec);
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t *out, int nranks, ncclUniqueId id, int rank) {
    if (bind_driver() || nranks < 1 || rank < 0 || rank >= nranks) return ncclInvalidArgument;
    ncclComm_t c = (ncclComm_t)calloc(1, sizeof *c);
    snprintf(c->name, sizeof c->name, "%s", id.internal);
    c->rank = rank;
    c->nranks = nranks;
    c->seg_bytes = sizeof(Hdr) + (size_t)nranks * SLOT_BYTES;
    int fd = -1;
    for (int tries = 0; tries < 200000 && fd < 0; ++tries) {
        fd = shm_open(c->name, O_RDWR | (rank == 0 ? O_CREAT : 0), 0600);
        if (fd < 0) usleep(100);
    }
    if (fd < 0) { free(c); return ncclSystemError; }
    if (rank == 0 && ftruncate(fd, (off_t)c->seg_bytes) != 0) { close(fd); free(c); return ncclSystemError; }
    struct stat st;
    for (int tries = 0; tries < 200000; ++tries) {  /* others wait until rank 0 sized it */
        if (fstat(fd, &st) == 0 && (size_t)st.st_size >= c->seg_bytes) break;
        usleep(100);
    }
    c->seg = (Hdr *)mmap(NULL, c->seg_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (c->seg == MAP_FAILED) { free(c); return ncclSystemError; }
    if (rank == 0) __atomic_store_n(&c->seg->nranks, nranks, __ATOMIC_RELEASE);
    while (__atomic_load_n(&c->seg->nranks, __ATOMIC_ACQUIRE) != nranks) sched_yield();
    c->tmp = (char *)malloc(SLOT_BYTES);
    barrier(c->seg);
    *out = c;
    return ncclSuccess;
}

static size_t dt_size(ncclDataType_t t) {
    switch (t) {
        case ncclInt8: case ncclUint8: return 1;
        case ncclFloat16: case ncclBfloat16: return 2;
        case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
        default: return 8;
    }
}

#define RED(T)                                                                          \
    do {                                                                                \
        T *a = (T *)acc;                                                                \
        const T *b = (const T *)in;                                                     \
        for (size_t i = 0; i < n; ++i)                                                  \
            a[i] = op == ncclSum ? (T)(a[i] + b[i]) : op == ncclProd ? (T)(a[i] * b[i]) \
                 : op == ncclMax ? (a[i] > b[i] ? a[i] : b[i]) : (a[i] < b[i] ? a[i] : b[i]); \
    } while (0)

static int reduce_into(char *acc, const char *in, size_t n, ncclDataType_t t, ncclRedOp_t op) {
    switch (t) {
        case ncclInt8: RED(int8_t); return 0;
        case ncclUint8: RED(uint8_t); return 0;
        case ncclInt32: RED(int32_t); return 0;
        case ncclUint32: RED(uint32_t); return 0;
        case ncclInt64: RED(int64_t); return 0;
        case ncclUint64: RED(uint64_t); return 0;
        case ncclFloat32: RED(float); return 0;
        case ncclFloat64: RED(double); return 0;
        default: return -1;
    }
}

ncclResult_t ncclAllReduce(const void *send, void *recv, size_t count, ncclDataType_t t, ncclRedOp_t op,
                           ncclComm_t c, cudaStream_t stream) {
    if (!c || op > ncclMin) return ncclInvalidArgument;
    const size_t es = dt_size(t), per = SLOT_BYTES / es;
    if (getenv("PGPCV_LOOPBACK_TRACE"))
        fprintf(stderr, "[loopback r%d] allreduce #%ld count %zu type %d op %d\n", c->rank, c->seq, count, (int)t, (int)op);
    ++c->seq;
    if (p_sync((void *)stream) != 0) return ncclUnhandledCudaError;
    for (size_t off = 0; off < count; off += per) {
        const size_t n = count - off < per ? count - off : per, bytes = n * es;
        if (p_d2h(slot(c, c->rank), (unsigned long long)(uintptr_t)((const char *)send + off * es), bytes,
                  (void *)stream) != 0 || p_sync((void *)stream) != 0)
            return ncclUnhandledCudaError;
        barrier(c->seg);
        memcpy(c->tmp, slot(c, 0), bytes);
        for (int r = 1; r < c->nranks; ++r)
            if (reduce_into(c->tmp, slot(c, r), n, t, op)) return ncclInvalidArgument;
        barrier(c->seg);
        if (p_h2d((unsigned long long)(uintptr_t)((char *)recv + off * es), c->tmp, bytes, (void *)stream) != 0 ||
            p_sync((void *)stream) != 0)
            return ncclUnhandledCudaError;
    }
    return ncclSuccess;
}

ncclResult_t ncclCommGetAsyncError(ncclComm_t c, ncclResult_t *err) {
    (void)c;
    *err = ncclSuccess;
    return ncclSuccess;
}

static ncclResult_t release(ncclComm_t c) {
    if (!c) return ncclSuccess;
    munmap(c->seg, c->seg_bytes);
    shm_unlink(c->name); /* every rank; later unlinks find it gone */
    free(c->tmp);
    free(c);
    return ncclSuccess;
}
ncclResult_t ncclCommDestroy(ncclComm_t c) { return release(c); }
ncclResult_t ncclCommAbort(ncclComm_t c) { return release(c); }
