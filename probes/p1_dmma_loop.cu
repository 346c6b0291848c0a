// P1 -- ceiling of the cv_kernel inner loop: DMMA.8x8x4 fed from shared memory in the
// kernel's exact fragment pattern (warp tile 16 x 64: per k-step 2 A + 8 B LDS.64 and
// 16 DMMA), with no global memory, at 1 and 2 CTAs of 8 warps per SM, and variants of the
// issue order.  Prints one JSON object (TFLOP/s per variant).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int AS = 132, BS = 68, KC = 16;

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

// variant 0: j outer / i inner (as cv_kernel); 1: i outer / j inner
template <int VAR>
__global__ void __launch_bounds__(256, 2) loop_kernel(double *out, int iters) {
    __shared__ __align__(16) double sm[KC * AS + KC * BS];
    for (int i = threadIdx.x; i < KC * AS + KC * BS; i += 256) sm[i] = 1e-3 * (i % 97);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
    double acc[2][8][2];
    for (int i = 0; i < 2; ++i) for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0;
    const double *As = sm, *Bs = sm + KC * AS;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k4 = 0; k4 < KC / 4; ++k4) {
            const double *ap = As + (k4 * 4 + t) * AS + warp * 16 + g;
            const double *bp = Bs + (k4 * 4 + t) * BS + g;
            double af[2], bf[8];
            af[0] = ap[0]; af[1] = ap[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) bf[j] = bp[j * 8];
            if (VAR == 0) {
#pragma unroll
                for (int j = 0; j < 8; ++j)
#pragma unroll
                    for (int i = 0; i < 2; ++i) dmma(acc[i][j], af[i], bf[j]);
            } else {
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) dmma(acc[i][j], af[i], bf[j]);
            }
        }
    }
    double s = 0;
    for (int i = 0; i < 2; ++i) for (int j = 0; j < 8; ++j) s += acc[i][j][0] + acc[i][j][1];
    if (s == 1234.5) out[0] = s;
}

template <typename F>
static double time_ms(F f) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    f(); CK(cudaDeviceSynchronize());
    cudaEventRecord(a); for (int r = 0; r < 5; ++r) f(); cudaEventRecord(b);
    CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms, a, b); return ms / 5;
}

int main() {
    cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
    double *out; CK(cudaMalloc(&out, 64));
    const int iters = 20000;
    printf("{\"sms\": %d", p.multiProcessorCount);
    for (int var = 0; var < 2; ++var)
        for (int cps = 1; cps <= 2; ++cps) {
            const int blocks = p.multiProcessorCount * cps;
            const double flop = (double)blocks * 8 * iters * (KC / 4) * 16 * 512.0;
            double ms = time_ms([&]() {
                if (var == 0) loop_kernel<0><<<blocks, 256>>>(out, iters);
                else loop_kernel<1><<<blocks, 256>>>(out, iters);
            });
            printf(", \"var%d_ctas%d_tflops\": %.3f", var, cps, flop / (ms * 1e-3) / 1e12);
        }
    printf("}\n");
    return 0;
}
