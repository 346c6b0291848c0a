// P7 -- FP64 DMMA throughput against the number of warps issuing it per SM sub-partition.
//
// The small-subset kernel runs 4 CTAs x 4 warps per SM (one warp of each CTA per SMSP) and
// only ~40 % of a CTA's time is spent in the update loop (profiles/r02_p2_c3_small_border.json),
// so on average ~1.5 warps per SMSP issue DMMA at any moment.  This probe measures what a
// given number of DMMA-issuing warps per SMSP can reach:
//   * W warps per SM (W / 4 per SMSP), each with NACC independent 8x8 accumulators;
//   * "reg": operands in registers (P0's loop); "lds": the small kernel's inner loop shape --
//     per k4 step 2 A + NACC/2 B fragments loaded from SMEM (LDS.64), NACC DMMAs.
// One JSON object on stdout: TFLOP/s per (variant, NACC, W).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <int NACC, bool LDS>
__global__ void k_dmma(double *out, int iters, double a_in, double b_in) {
    __shared__ double sm[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = 1e-3 * (i & 63);
    __syncthreads();
    double c[NACC][2];
#pragma unroll
    for (int j = 0; j < NACC; ++j) c[j][0] = c[j][1] = 0.0;
    const double a0 = a_in + threadIdx.x * 1e-9, b0 = b_in - threadIdx.x * 1e-9;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double *ap = sm + (warp & 3) * 256 + (lane >> 2) * 16 + (lane & 3);
    const double *bp = sm + 1024 + (lane >> 2) * 16 + (lane & 3);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) {
            if constexpr (LDS) {
                const int o = (k4 << 2) ^ (((lane >> 2) & 3) << 2);
                double af[2], bf[NACC / 2];
                af[0] = ap[o];
                af[1] = ap[128 + o];
#pragma unroll
                for (int j = 0; j < NACC / 2; ++j) bf[j] = bp[j * 128 + o];
#pragma unroll
                for (int j = 0; j < NACC / 2; ++j)
#pragma unroll
                    for (int h = 0; h < 2; ++h) dmma(c[j * 2 + h], af[h], bf[j]);
            } else {
#pragma unroll
                for (int j = 0; j < NACC; ++j) dmma(c[j], a0, b0);
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < NACC; ++j) s += c[j][0] + c[j][1];
    if (s == 12345.678) out[blockIdx.x] = s;
}

template <int NACC, bool LDS>
static double run(int sms, int warps_per_sm, double *out) {
    // one CTA per SM of warps_per_sm warps (the warps spread over the 4 SMSPs round-robin)
    const int threads = 32 * warps_per_sm;
    const int iters = 2048 * 8 / NACC;
    const double flop = (double)sms * warps_per_sm * iters * 4 * NACC * (8.0 * 8 * 4 * 2);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    k_dmma<NACC, LDS><<<sms, threads>>>(out, iters, 0.999999, 1e-7);
    CK(cudaDeviceSynchronize());
    const int reps = 20;
    CK(cudaEventRecord(e0));
    for (int r = 0; r < reps; ++r) k_dmma<NACC, LDS><<<sms, threads>>>(out, iters, 0.999999, 1e-7);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    CK(cudaGetLastError());
    return flop * reps / (ms * 1e-3) / 1e12;
}

int main() {
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, 0));
    double *out;
    CK(cudaMalloc(&out, 1 << 20));
    const int sms = p.multiProcessorCount;
    const int ws[] = {4, 8, 12, 16, 32};
    printf("{\"sms\": %d", sms);
    for (int w : ws) {
        printf(", \"reg_n8_w%d\": %.2f", w, run<8, false>(sms, w, out));
        printf(", \"reg_n16_w%d\": %.2f", w, run<16, false>(sms, w, out));
        printf(", \"lds_n8_w%d\": %.2f", w, run<8, true>(sms, w, out));
        printf(", \"lds_n16_w%d\": %.2f", w, run<16, true>(sms, w, out));
        printf(", \"lds_n32_w%d\": %.2f", w, run<32, true>(sms, w, out));
    }
    printf("}\n");
    return 0;
}
