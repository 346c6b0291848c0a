// P0 — FP64 peak probe for B200 (sm_100a).
//
// Measures the two FP64 instruction paths the Cholesky kernel can use:
//   * DFMA  (plain FP64 FMA on the CUDA-core FP64 pipe)
//   * DMMA  (mma.sync.aligned.m8n8k4 .f64 -> SASS DMMA.8x8x4, the FP64 tensor path)
// each as a short burst (~0.2 s) and sustained (~4 s back to back), with CUDA events.
// Prints one JSON object on stdout.  This is the denominator the bench reports
// "% of measured FP64 peak" against.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

// 8 independent FMA chains per thread; iters * 8 * 2 flop per thread.
__global__ void dfma_kernel(double *out, int iters, double a, double b) {
    double r0 = threadIdx.x, r1 = r0 + 1, r2 = r0 + 2, r3 = r0 + 3;
    double r4 = r0 + 4, r5 = r0 + 5, r6 = r0 + 6, r7 = r0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            r0 = fma(r0, a, b); r1 = fma(r1, a, b); r2 = fma(r2, a, b); r3 = fma(r3, a, b);
            r4 = fma(r4, a, b); r5 = fma(r5, a, b); r6 = fma(r6, a, b); r7 = fma(r7, a, b);
        }
    }
    double s = r0 + r1 + r2 + r3 + r4 + r5 + r6 + r7;
    if (s == 12345.678) out[blockIdx.x] = s;  // keep the chains alive
}

// Each warp: 8 independent 8x8 accumulators, one m8n8k4 DMMA each per inner step.
__global__ void dmma_kernel(double *out, int iters, double a_in, double b_in) {
    double a = a_in + threadIdx.x * 1e-9, b = b_in - threadIdx.x * 1e-9;
    double c[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) { c[j][0] = 0.0; c[j][1] = 0.0; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
    if (s == 12345.678) out[blockIdx.x] = s;
}

static int g_sms = 0;

template <typename F>
static double time_ms(F launch, int reps) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    launch();  // warm-up
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int r = 0; r < reps; ++r) launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0; CK(cudaEventElapsedTime(&ms, e0, e1));
    CK(cudaGetLastError());
    return ms;
}

int main(int argc, char **argv) {
    double sustain_s = argc > 1 ? atof(argv[1]) : 4.0;
    cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
    g_sms = p.multiProcessorCount;
    int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    double *out; CK(cudaMalloc(&out, 1 << 20));

    printf("{\"gpu\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\", \"clock_rate_khz\": %d, \"l2_bytes\": %d, "
           "\"smem_optin_per_block\": %zu, \"regs_per_sm\": %d", p.name, g_sms, p.major, p.minor, clk_khz,
           p.l2CacheSize, p.sharedMemPerBlockOptin, p.regsPerMultiprocessor);

    // DFMA: blocks = sms * 8, threads 256 (8 warps/block -> 64 warps/SM).
    for (int variant = 0; variant < 2; ++variant) {
        const char *name = variant == 0 ? "dfma" : "dmma";
        int blocks = g_sms * (variant == 0 ? 8 : 4);
        int threads = 256;
        int iters = variant == 0 ? 2048 : 1024;
        double flop_per_launch = variant == 0
            ? (double)blocks * threads * iters * 16 * 8 * 2
            : (double)blocks * (threads / 32) * iters * 4 * 8 * (8.0 * 8 * 4 * 2);
        auto launch = [&]() {
            if (variant == 0) dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
            else dmma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        };
        // calibrate
        double ms1 = time_ms(launch, 3) / 3;
        int reps_burst = (int)(200.0 / ms1) + 1;
        double ms_b = time_ms(launch, reps_burst);
        double tf_burst = flop_per_launch * reps_burst / (ms_b * 1e-3) / 1e12;
        int reps_sus = (int)(sustain_s * 1000.0 / ms1) + 1;
        double ms_s = time_ms(launch, reps_sus);
        double tf_sus = flop_per_launch * reps_sus / (ms_s * 1e-3) / 1e12;
        printf(", \"%s_tflops_burst\": %.3f, \"%s_tflops_sustained\": %.3f, \"%s_ms_per_launch\": %.3f",
               name, tf_burst, name, tf_sus, name, ms1);
    }
    printf("}\n");
    return 0;
}
