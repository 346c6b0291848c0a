// P5 -- the cv_kernel update loop in isolation: persistent CTAs (2 per SM, 8 warps, warp tile
// 16 x 64) stream operand chunks (A: 128 x 16, B: 64 x 16 doubles = 24 KB) from global
// memory into 3 SMEM stages with cp.async.bulk + full/empty mbarriers, exactly the
// cv_kernel protocol (producer = thread 0 after the empty wait, consumer-side
// fence.proxy.async before each release, L2 prefetch PFD chunks ahead), and run the same
// DMMA fragment pattern.  No generation, no diagonal block, no TRSM.
//
// Questions: (1) how close the protocol alone comes to the P1 inner-loop ceiling (36.4
// TFLOP/s); (2) whether streaming from DRAM (operands spread over a buffer far larger than
// L2) costs throughput against operands that hit in L2 (a small buffer); (3) power, sampled
// by the driver script while each variant runs for `seconds`.
//
//   p5_stream <buffer_MB> <seconds> [b_shared]
//     buffer_MB: operand footprint (e.g. 32 -> L2-resident, 16384 -> DRAM-streamed)
//     b_shared:  1 = the two CTAs of a pair read the same B chunks (emulates a pair sharing
//                the B panel through L2), 0 = independent B streams (as cv_kernel)
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int MT = 128, NB = 64, KC = 16, NT = 256, NWARP = 8, STAGES = 3, PFD = 4;
constexpr int A_STAGE = MT * KC, B_STAGE = NB * KC;
constexpr unsigned STAGE_BYTES = (A_STAGE + B_STAGE) * 8;

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned par) {
    unsigned done = 0;
    do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(smem_u32(b)), "r"(par) : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void *p, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

// chunk n of CTA c: A and B addresses inside the buffer (wrapping), 24 KB apart per chunk
__device__ __forceinline__ const double *a_src(const double *buf, size_t nchunk, int cta, long n) {
    return buf + ((size_t)(cta * 7919L + n) % nchunk) * (A_STAGE + B_STAGE);
}
__device__ __forceinline__ const double *b_src(const double *buf, size_t nchunk, int cta, long n, int shared) {
    const int owner = shared ? (cta & ~1) : cta;
    return buf + ((size_t)(owner * 7919L + n) % nchunk) * (A_STAGE + B_STAGE) + A_STAGE;
}

__global__ void __launch_bounds__(NT, 2) stream_kernel(const double *buf, size_t nchunk, long chunks, int shared,
                                                       double *out) {
    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
    if (tid == 0) {
        for (int i = 0; i < STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], NWARP); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](long n) {
        const int s = n % STAGES;
        const long use = n / STAGES;
        if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
        double *sb = smem + s * (A_STAGE + B_STAGE);
        mbar_expect_tx(&full[s], STAGE_BYTES);
        bulk_g2s(sb, a_src(buf, nchunk, blockIdx.x, n), A_STAGE * 8, &full[s]);
        bulk_g2s(sb + A_STAGE, b_src(buf, nchunk, blockIdx.x, n, shared), B_STAGE * 8, &full[s]);
    };
    if (tid == 0) {
        asm volatile("fence.proxy.async.global;\n fence.proxy.async.shared::cta;" ::: "memory");
        for (long i = 0; i < STAGES - 1 && i < chunks; ++i) issue(i);
        for (long i = STAGES - 1; i < STAGES - 1 + PFD && i < chunks; ++i) {
            prefetch_l2(a_src(buf, nchunk, blockIdx.x, i), A_STAGE * 8);
            prefetch_l2(b_src(buf, nchunk, blockIdx.x, i, shared), B_STAGE * 8);
        }
    }
    __syncwarp();
    double acc[2][8][2];
    for (int i = 0; i < 2; ++i) for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int sw = (g & 3) << 2;
    for (long n = 0; n < chunks; ++n) {
        if (tid == 0) {
            if (n + STAGES - 1 < chunks) issue(n + STAGES - 1);
            if (n + STAGES - 1 + PFD < chunks) {
                prefetch_l2(a_src(buf, nchunk, blockIdx.x, n + STAGES - 1 + PFD), A_STAGE * 8);
                prefetch_l2(b_src(buf, nchunk, blockIdx.x, n + STAGES - 1 + PFD, shared), B_STAGE * 8);
            }
        }
        mbar_wait(&full[n % STAGES], (n / STAGES) & 1);
        __syncwarp();
        const double *As = smem + (n % STAGES) * (A_STAGE + B_STAGE);
        const double *ap = As + (warp * 16 + g) * KC + t;
        const double *bp = As + A_STAGE + g * KC + t;
#pragma unroll
        for (int k4 = 0; k4 < KC / 4; ++k4) {
            const int o = (k4 << 2) ^ sw;
            double af[2], bf[8];
            af[0] = ap[o];
            af[1] = ap[8 * KC + o];
#pragma unroll
            for (int j = 0; j < 8; ++j) bf[j] = bp[j * 8 * KC + o];
#pragma unroll
            for (int j = 0; j < 8; ++j)
#pragma unroll
                for (int i = 0; i < 2; ++i) dmma(acc[i][j], af[i], bf[j]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[n % STAGES]);
    }
    double s = 0;
    for (int i = 0; i < 2; ++i) for (int j = 0; j < 8; ++j) s += acc[i][j][0] + acc[i][j][1];
    if (s == 1234.5) out[0] = s;
}

int main(int argc, char **argv) {
    const size_t mb = argc > 1 ? atol(argv[1]) : 32;
    const double seconds = argc > 2 ? atof(argv[2]) : 4.0;
    const int shared = argc > 3 ? atoi(argv[3]) : 0;
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, 0));
    const size_t chunk_bytes = (size_t)(A_STAGE + B_STAGE) * 8;
    const size_t nchunk = mb * 1024 * 1024 / chunk_bytes;
    double *buf, *out;
    CK(cudaMalloc(&buf, nchunk * chunk_bytes));
    CK(cudaMemset(buf, 0, nchunk * chunk_bytes));
    CK(cudaMalloc(&out, 64));
    const size_t smem = (size_t)STAGES * STAGE_BYTES;
    CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int blocks = 2 * p.multiProcessorCount;
    long chunks = 2000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    // calibrate one launch to ~0.5 s, then repeat for `seconds`
    stream_kernel<<<blocks, NT, smem>>>(buf, nchunk, chunks, shared, out);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    stream_kernel<<<blocks, NT, smem>>>(buf, nchunk, chunks, shared, out);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    chunks = (long)(chunks * 500.0 / ms);
    const int reps = (int)(seconds / 0.5) + 1;
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) stream_kernel<<<blocks, NT, smem>>>(buf, nchunk, chunks, shared, out);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    const double flop = (double)reps * blocks * NWARP * chunks * (KC / 4) * 16 * 512.0;
    printf("{\"buffer_mb\": %zu, \"b_shared\": %d, \"seconds\": %.2f, \"tflops\": %.3f, \"dram_or_l2_TBps\": %.3f}\n",
           mb, shared, ms / 1e3, flop / (ms * 1e-3) / 1e12,
           (double)reps * blocks * chunks * chunk_bytes / (ms * 1e-3) / 1e12);
    return 0;
}
