// P6 -- variants of the cv_kernel operand pipeline, in isolation (P5 showed the update loop
// alone, with the round-1 protocol, reaches 30.6 TFLOP/s from DRAM against the 36.4 of the
// SMEM-only P1 loop: the protocol, not the non-GEMM phases, bounds the large kernel).
// Each variant: persistent CTAs, 2 per SM, 8 compute warps with a 16 x 64 warp tile
// (128 x 64 CTA tile), operands streamed from a buffer far larger than L2.
//   KC      k-columns per stage (16: one column group; 32: two, 4 bulk copies per stage)
//   STAGES  SMEM ring depth
//   FENCE   consumer-side fence.proxy.async.shared::cta before releasing a stage
//   PROD    0: thread 0 of warp 0 produces (round 1); 1: a 9th warp only produces
//   SPLIT   1: two half-stage barriers (A/B of the k-columns 0-7 and 8-15 land separately
//           and the warps start on the first half) -- only with KC = 16
// Usage: p6_protocol <variant 0..N-1 | -1 all> <seconds> [buffer_MB]; one JSON line per run.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int MT = 128, NB = 64, NWARP = 8, PFD = 4;

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

// A group chunk: MT x 16 doubles (16 KB); B: NB x 16 (8 KB); a "unit" = one 16-column group
constexpr int AG = MT * 16, BG = NB * 16, UNIT = AG + BG;

template <int KC, int STAGES, int FENCE, int PROD, int SPLIT, int LAST = 0, int PF2 = 0, int WB = 0>
__global__ void __launch_bounds__(32 * (NWARP + PROD), 2) proto_kernel(const double *buf, size_t nunits, long chunks,
                                                                        double *out) {
    // KC = 8: 8-column groups (64-B rows; the swizzle moves rows 2-3 of every 4 to the other
    // half-row, conflict-free fragment loads); KC >= 16: KC / 16 groups of 16 columns per stage
    constexpr int W = KC < 16 ? KC : 16;
    constexpr int AG = MT * W, BG = NB * W, UNIT = AG + BG;
    constexpr int G = KC / W;  // column groups per stage
    constexpr int STAGE = G * UNIT;
    constexpr int NBAR = SPLIT ? 2 : 1;
    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) uint64_t full[STAGES * NBAR], empty[STAGES];
    __shared__ unsigned rel[STAGES];  // LAST: releases of the stage's current use
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
    if (tid == 0) {
        for (int i = 0; i < STAGES * NBAR; ++i) mbar_init(&full[i], 1);
        for (int i = 0; i < STAGES; ++i) mbar_init(&empty[i], NWARP);
        for (int i = 0; i < STAGES; ++i) rel[i] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto src = [&](long n, int gi) { return buf + ((size_t)(blockIdx.x * 7919L + n * G + gi) % nunits) * UNIT; };
    auto issue = [&](long n) {
        const int s = n % STAGES;
        const long use = n / STAGES;
        if (!LAST && use > 0) mbar_wait(&empty[s], (use - 1) & 1);
        double *sb = smem + s * STAGE;
        if (SPLIT) {  // k-columns 0-7 and 8-15 of the group as two halves (A rows x 8 each)
            // emulate: two bulk copies per half (the data layout is irrelevant for timing)
            mbar_expect_tx(&full[s * 2], UNIT * 4);
            bulk_g2s(sb, src(n, 0), AG * 4, &full[s * 2]);
            bulk_g2s(sb + AG, src(n, 0) + AG, BG * 4, &full[s * 2]);
            mbar_expect_tx(&full[s * 2 + 1], UNIT * 4);
            bulk_g2s(sb + AG / 2, src(n, 0) + AG / 2, AG * 4, &full[s * 2 + 1]);
            bulk_g2s(sb + AG + BG / 2, src(n, 0) + AG + BG / 2, BG * 4, &full[s * 2 + 1]);
        } else {
            mbar_expect_tx(&full[s], STAGE * 8);
            for (int gi = 0; gi < G; ++gi) {
                bulk_g2s(sb + gi * UNIT, src(n, gi), AG * 8, &full[s]);
                bulk_g2s(sb + gi * UNIT + AG, src(n, gi) + AG, BG * 8, &full[s]);
            }
        }
    };
    auto pref = [&](long n) {
        for (int gi = 0; gi < G; ++gi) {
            if (PF2) {  // A and B separately, as cv_kernel (its A and B chunks are apart)
                prefetch_l2(src(n, gi), AG * 8);
                prefetch_l2(src(n, gi) + AG, BG * 8);
            } else {
                prefetch_l2(src(n, gi), UNIT * 8);
            }
        }
    };
    if (PROD && warp == NWARP) {  // the producer warp
        if (lane == 0) {
            asm volatile("fence.proxy.async.global;\n fence.proxy.async.shared::cta;" ::: "memory");
            for (long n = 0; n < chunks; ++n) {
                issue(n);
                if (n + PFD < chunks) pref(n + PFD);
            }
        }
        return;
    }
    if (!PROD && tid == 0) {
        asm volatile("fence.proxy.async.global;\n fence.proxy.async.shared::cta;" ::: "memory");
        const int pro = LAST ? STAGES : STAGES - 1;
        for (long i = 0; i < pro && i < chunks; ++i) issue(i);
        for (long i = pro; i < pro + PFD && i < chunks; ++i) pref(i);
    }
    __syncwarp();
    double acc[2][8][2];
    for (int i = 0; i < 2; ++i) for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int sw = W == 16 ? (g & 3) << 2 : ((g >> 1) & 1) << 2;
    for (long n = 0; n < chunks; ++n) {
        if (!PROD && !LAST && tid == 0) {
            if (n + STAGES - 1 < chunks) issue(n + STAGES - 1);
            if (n + STAGES - 1 + PFD < chunks) pref(n + STAGES - 1 + PFD);
        }
        const int s = n % STAGES;
        const unsigned par = (n / STAGES) & 1;
        if (WB) {  // wait before the fragment loop, as cv_kernel
            mbar_wait(&full[s], par);
            __syncwarp();
        }
#pragma unroll
        for (int gi = 0; gi < G; ++gi) {
            const double *As = smem + s * STAGE + gi * UNIT;
            const double *ap = As + (warp * 16 + g) * W + t;
            const double *bp = As + AG + g * W + t;
#pragma unroll
            for (int k4 = 0; k4 < W / 4; ++k4) {
                if (!WB && (SPLIT ? (k4 == 0 || k4 == 2) : (gi == 0 && k4 == 0))) {
                    mbar_wait(&full[SPLIT ? s * 2 + (k4 >> 1) : s], par);
                    __syncwarp();
                }
                const int o = (k4 << 2) ^ sw;
                double af[2], bf[8];
                af[0] = ap[o];
                af[1] = ap[8 * W + o];
#pragma unroll
                for (int j = 0; j < 8; ++j) bf[j] = bp[j * 8 * W + o];
#pragma unroll
                for (int j = 0; j < 8; ++j)
#pragma unroll
                    for (int i = 0; i < 2; ++i) dmma(acc[i][j], af[i], bf[j]);
            }
        }
        if (FENCE) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (LAST) {
            // the last warp to release stage s refills it with chunk n + STAGES
            if (lane == 0) {
                unsigned old;
                asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(smem_u32(&rel[s])) : "memory");
                if (old == NWARP - 1) {
                    rel[s] = 0;
                    if (n + STAGES < chunks) issue(n + STAGES);
                    if (n + STAGES + PFD < chunks) pref(n + STAGES + PFD);
                }
            }
            __syncwarp();
        } else if (lane == 0) {
            mbar_arrive(&empty[s]);
        }
    }
    double sum = 0;
    for (int i = 0; i < 2; ++i) for (int j = 0; j < 8; ++j) sum += acc[i][j][0] + acc[i][j][1];
    if (sum == 1234.5) out[0] = sum;
}

struct Variant {
    const char *name;
    int kc, stages, fence, prod, split;
    void (*launch)(int, size_t, const double *, size_t, long, double *);
};

template <int KC, int ST, int F, int P, int S, int LA, int PF2, int WB>
void launch_v(int blocks, size_t smem, const double *buf, size_t nunits, long chunks, double *out) {
    proto_kernel<KC, ST, F, P, S, LA, PF2, WB><<<blocks, 32 * (NWARP + P), smem>>>(buf, nunits, chunks, out);
}
template <int KC, int ST, int F, int P, int S, int LA = 0, int PF2 = 0, int WB = 0>
Variant mk(const char *name) {
    CK(cudaFuncSetAttribute(proto_kernel<KC, ST, F, P, S, LA, PF2, WB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            ST * KC * (MT + NB) * 8));
    return Variant{name, KC, ST, F, P, S, launch_v<KC, ST, F, P, S, LA, PF2, WB>};
}

int main(int argc, char **argv) {
    const int which = argc > 1 ? atoi(argv[1]) : -1;
    const double seconds = argc > 2 ? atof(argv[2]) : 3.0;
    const size_t mb = argc > 3 ? atol(argv[3]) : 4096;
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, 0));
    const size_t nunits = mb * 1024 * 1024 / (UNIT * 8);
    double *buf, *out;
    CK(cudaMalloc(&buf, nunits * UNIT * 8));
    CK(cudaMemset(buf, 0, nunits * UNIT * 8));
    CK(cudaMalloc(&out, 64));
    Variant vs[] = {
        mk<16, 3, 1, 0, 0>("round1: KC16 S3 fence, thread-0 producer"),
        mk<16, 3, 0, 0, 0>("KC16 S3 no fence"),
        mk<16, 4, 1, 0, 0>("KC16 S4 fence"),
        mk<32, 2, 1, 0, 0>("KC32 S2 fence"),
        mk<16, 3, 1, 1, 0>("KC16 S3 fence, producer warp"),
        mk<16, 4, 1, 1, 0>("KC16 S4 fence, producer warp"),
        mk<16, 4, 0, 1, 0>("KC16 S4 no fence, producer warp"),
        mk<16, 3, 1, 0, 1>("KC16 S3 fence, split half-stage barriers"),
        mk<16, 3, 1, 0, 0, 1>("KC16 S3 fence, last releasing warp refills"),
        mk<16, 4, 1, 0, 0, 1>("KC16 S4 fence, last releasing warp refills"),
        mk<32, 2, 1, 0, 0, 1>("KC32 S2 fence, last releasing warp refills"),
        mk<16, 3, 1, 0, 0, 0, 1, 0>("round1 + A/B prefetched separately"),
        mk<16, 3, 1, 0, 0, 0, 0, 1>("round1 + wait before the fragment loop"),
        mk<16, 3, 1, 0, 0, 0, 1, 1>("round1 + both (= cv_kernel / P5 structure)"),
        mk<8, 6, 1, 0, 0, 0, 1, 1>("KC8 S6 fence (72 KB), thread-0 producer, cv_kernel structure"),
        mk<8, 7, 1, 0, 0, 0, 1, 1>("KC8 S7 fence (84 KB), thread-0 producer, cv_kernel structure"),
        mk<8, 6, 0, 0, 0, 0, 1, 1>("KC8 S6 no fence, thread-0 producer, cv_kernel structure"),
        mk<16, 3, 0, 0, 0, 0, 1, 1>("KC16 S3 no fence, cv_kernel structure"),
        mk<8, 6, 1, 0, 0, 1, 1, 1>("KC8 S6 fence, last releasing warp refills"),
    };
    const int nv = sizeof(vs) / sizeof(vs[0]);
    const int blocks = 2 * p.multiProcessorCount;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int v = 0; v < nv; ++v) {
        if (which >= 0 && v != which) continue;
        const Variant &V = vs[v];
        const size_t smem = (size_t)V.stages * V.kc * (MT + NB) * 8;
        long chunks = 400 * 16 / V.kc;
        V.launch(blocks, smem, buf, nunits, chunks, out);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        V.launch(blocks, smem, buf, nunits, chunks, out);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        chunks = (long)(chunks * 400.0 / ms);
        const int reps = (int)(seconds / 0.4) + 1;
        cudaEventRecord(a);
        for (int r = 0; r < reps; ++r) V.launch(blocks, smem, buf, nunits, chunks, out);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        CK(cudaGetLastError());
        cudaEventElapsedTime(&ms, a, b);
        const double flop = (double)reps * blocks * NWARP * chunks * (V.kc / 4) * 16 * 512.0;
        printf("{\"variant\": %d, \"name\": \"%s\", \"smem_kb\": %.1f, \"tflops\": %.3f, \"seconds\": %.2f}\n", v,
               V.name, smem / 1024.0, flop / (ms * 1e-3) / 1e12, ms / 1e3);
        fflush(stdout);
    }
    return 0;
}
