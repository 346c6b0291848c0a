// cv_kernel.cu -- the hot path of parallel cross-validation on B200 (sm_100a), FP64.
//
// One persistent CTA per factorization slot pulls (subset s, config c) work items in LPT
// order and, for each, evaluates the subset's local SSPE z_i of Alg.1 line 7 (PAPER.md
// P:224) exactly as Eq.3/Eq.4 define it:
//
//   A  = Sigma(theta) + lambda I,  Sigma_ij = exp(-||t_i - t_j|| / theta)
//   A  = L L^T                      blocked left-looking Cholesky (FP64)
//   z  = L^{-1} y_T                 fused: y_T^T is a bordered extra row of A
//   alpha = L^{-T} z                blocked backward substitution
//   yhat_v = sum_j c(v, t_j) alpha_j,  z_i = sum_v (yhat_v - y_v)^2        (Eq.3, Eq.4)
//
// Nothing is precomputed per config: every entry of A, of the bordered row and of the
// cross-covariance is generated where it is consumed, from the subset's staged
// coordinates (distance -> exp), so a config costs no HBM traffic beyond the factor L.
//
// Data layout (per resident CTA, in HBM): L is column-major with leading dimension
// ld = roundup(k+1, 16) doubles; rows 0..k-1 hold the Cholesky factor, row k holds z.
//
// Left-looking step for block column j (width NB = 64, columns j0..j0+jw-1), for every
// row tile of MT = 128 rows r0.. (rows j0..k):
//   acc    = L[r0:r0+MT, 0:j0] . L[j0:j0+NB, 0:j0]^T       -- FP64 DMMA (mma.m8n8k4),
//            operands streamed HBM/L2 -> SMEM by a 3-stage cp.async pipeline, KC = 32
//   C      = A[r0:r0+MT, j0:j0+NB] - acc                    -- generated on the fly
//   tile 0 : L_jj = chol(C[0:jw, 0:jw]) and Linv = L_jj^{-1}, fused, in SMEM
//   X      = C . Linv^T                                      -- FP64 DMMA (TRSM as GEMM)
//   L[r0:, j0:j0+jw] = X   (tile 0: its first jw rows are L_jj itself)
//
// SMEM operand tiles are k-major with a row stride of MT+4 / NB+4 doubles: a stride of
// 8 (mod 32) 4-byte words makes the DMMA A/B fragment loads (lane (g,t) reads element
// [t][g]) conflict-free per half-warp.
#include <cmath>
#include <cstdint>

#include "pgpcv_internal.h"

namespace pgpcv {
namespace {

constexpr int MT = kMT;
constexpr int NB = kNB;
constexpr int NT = kThreads;
constexpr int KC = 32;
constexpr int STAGES = 3;
constexpr int AS = MT + 4;  // 132 doubles = 264 words == 8 (mod 32)
constexpr int BS = NB + 4;  // 68 doubles  = 136 words == 8 (mod 32)
constexpr int LJS = NB + 1; // 65: odd stride for the back-substitution diagonal block
constexpr int A_STAGE = KC * AS;
constexpr int B_STAGE = KC * BS;
constexpr int STAGE_DBL = STAGES * (A_STAGE + B_STAGE); // 19,200 doubles
constexpr int CS_DBL = NB * AS;                         // C tile, aliases the stages
constexpr int BT_DBL = NB * BS;                         // Linv^T tile
constexpr int COORD_DBL = 2 * MT + 3 * NB;
constexpr int MISC_DBL = NB + 16;
constexpr size_t SMEM_BYTES = sizeof(double) * (STAGE_DBL + BT_DBL + COORD_DBL + MISC_DBL);
static_assert(CS_DBL <= STAGE_DBL, "C tile must fit in the stage buffers");
static_assert(NB * LJS <= BT_DBL, "back-substitution block must fit in the Linv buffer");
static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
static_assert((AS * 2) % 32 == 8 && (BS * 2) % 32 == 8, "fragment-load strides");
static_assert(MT == 4 * 32 && NB == 2 * 32 && NT == 256, "8 warps as 4 (M) x 2 (N), 32x32 each");

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, int src_bytes) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// D = A(8x4, row) * B(4x8, col) + D on the FP64 tensor path (SASS DMMA.8x8x4).
// Fragments: a = A[g][t], b = B[t][g], d = {D[g][2t], D[g][2t+1]} for lane = 4g + t.
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d[0]), "+d"(d[1])
        : "d"(a), "d"(b));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Stage KC columns (kk..kk+KC-1) of two row ranges of L into SMEM, k-major:
//   As[q][rr] = L[r0 + rr, kk + q]  (rows >= nva zero-filled)
//   Bs[q][rr] = L[j0 + rr, kk + q]  (rows >= nvb zero-filled)
__device__ __forceinline__ void load_stage(double *As, double *Bs, const double *L, int64_t ld,
                                           int r0, int nva, int j0, int nvb, int kk, int tid) {
#pragma unroll
    for (int i = 0; i < (KC * MT / 2) / NT; ++i) {
        const int e = tid + i * NT;
        const int q = e / (MT / 2);
        const int rr = (e % (MT / 2)) * 2;
        const int row = r0 + rr;
        const int nbytes = row + 2 <= nva ? 16 : (row < nva ? 8 : 0);
        const double *src = nbytes ? L + (size_t)(kk + q) * ld + row : L;
        cp_async16(As + q * AS + rr, src, nbytes);
    }
#pragma unroll
    for (int i = 0; i < (KC * NB / 2) / NT; ++i) {
        const int e = tid + i * NT;
        const int q = e / (NB / 2);
        const int rr = (e % (NB / 2)) * 2;
        const int row = j0 + rr;
        const int nbytes = row + 2 <= nvb ? 16 : (row < nvb ? 8 : 0);
        const double *src = nbytes ? L + (size_t)(kk + q) * ld + row : L;
        cp_async16(Bs + q * BS + rr, src, nbytes);
    }
}

// acc[i][j] += A[wm*32 + 8i .., k] * B[k, wn*32 + 8j ..] over ksteps*4 values of k, with
// A stored k-major at stride as and B stored k-major at stride bs.
template <int KSTEPS>
__device__ __forceinline__ void mma_tile(double (&acc)[4][4][2], const double *As, int as,
                                         const double *Bs, int bs, int wm, int wn, int g, int t) {
#pragma unroll
    for (int k4 = 0; k4 < KSTEPS; ++k4) {
        const double *ap = As + (k4 * 4 + t) * as + wm * 32 + g;
        const double *bp = Bs + (k4 * 4 + t) * bs + wn * 32 + g;
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = ap[i * 8];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = bp[j * 8];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
    }
}

__global__ void __launch_bounds__(NT, 1) cv_kernel(CvArgs a) {
    extern __shared__ __align__(16) double smem[];
    double *stage = smem;
    double *Cs = smem;                  // aliases the stages after the update GEMM
    double *Bt = smem + STAGE_DBL;      // Bt[q*BS + n] = Linv[n][q]
    double *rx = Bt + BT_DBL;           // row-tile coordinates
    double *ry = rx + MT;
    double *cx = ry + MT;               // block-column coordinates and values
    double *cy = cx + NB;
    double *cv = cy + NB;
    double *dg = cv + NB;               // sqrt pivots of the diagonal block
    double *red = dg + NB;              // per-warp partial sums
    __shared__ int s_item;
    __shared__ int s_fail;

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp & 3, wn = warp >> 2;
    double *L = a.work + (size_t)blockIdx.x * a.slot_stride;

    for (;;) {
        if (tid == 0) s_item = (int)atomicAdd(a.counter, 1u);
        __syncthreads();
        const int item = s_item;
        __syncthreads();
        if (item >= a.n_items) break;
        const int s = a.items[item].x;
        const int c = a.items[item].y;
        const int64_t toff = a.train_off[s];
        const int k = (int)(a.train_off[s + 1] - toff);
        const int64_t voff = a.val_off[s];
        const int m = (int)(a.val_off[s + 1] - voff);
        const double *tx = a.tx + toff, *ty = a.ty + toff, *tv = a.tv + toff;
        const double range = a.params[3 * c], sigma2 = a.params[3 * c + 1];
        const double nugget = a.params[3 * c + 2];
        const double lam = nugget / sigma2;
        const double ninv = -1.0 / range;
        const int64_t ld = factor_ld(k);
        const int nblk = (k + NB - 1) / NB;
        bool failed = false;

        // ---------------- blocked left-looking Cholesky with bordered y row ----------------
        for (int jb = 0; jb < nblk && !failed; ++jb) {
            const int j0 = jb * NB;
            const int jw = min(NB, k - j0);
            const int nrows = k + 1 - j0;  // rows j0..k (row k: bordered y)
            const int ntiles = (nrows + MT - 1) / MT;
            for (int i = tid; i < NB; i += NT) {
                const int cc = j0 + i;
                const bool ok = cc < k;
                cx[i] = ok ? __ldg(tx + cc) : 0.0;
                cy[i] = ok ? __ldg(ty + cc) : 0.0;
                cv[i] = ok ? __ldg(tv + cc) : 0.0;
            }
            for (int rt = 0; rt < ntiles; ++rt) {
                const int r0 = j0 + rt * MT;
                for (int i = tid; i < MT; i += NT) {
                    const int r = r0 + i;
                    rx[i] = r < k ? __ldg(tx + r) : 0.0;
                    ry[i] = r < k ? __ldg(ty + r) : 0.0;
                }
                double acc[4][4][2];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

                // acc = L[r0:r0+MT, 0:j0] . L[j0:j0+NB, 0:j0]^T
                const int nk = j0 / KC;
                if (nk > 0) {
#pragma unroll
                    for (int st = 0; st < STAGES - 1; ++st) {
                        if (st < nk)
                            load_stage(stage + st * (A_STAGE + B_STAGE),
                                       stage + st * (A_STAGE + B_STAGE) + A_STAGE, L, ld, r0,
                                       k + 1, j0, k, st * KC, tid);
                        cp_async_commit();
                    }
                    for (int kc = 0; kc < nk; ++kc) {
                        cp_async_wait<STAGES - 2>();
                        __syncthreads();
                        const int nxt = kc + STAGES - 1;
                        if (nxt < nk) {
                            double *sb = stage + (nxt % STAGES) * (A_STAGE + B_STAGE);
                            load_stage(sb, sb + A_STAGE, L, ld, r0, k + 1, j0, k, nxt * KC, tid);
                        }
                        cp_async_commit();
                        const double *As = stage + (kc % STAGES) * (A_STAGE + B_STAGE);
                        mma_tile<KC / 4>(acc, As, AS, As + A_STAGE, BS, wm, wn, g, t);
                    }
                    cp_async_wait<0>();
                }
                __syncthreads();

                // C = A - acc, A generated on the fly (Eq.3 second line)
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int ml = wm * 32 + i * 8 + g;
                            const int nl = wn * 32 + j * 8 + 2 * t + e;
                            const int r = r0 + ml, cc = j0 + nl;
                            double av;
                            if (cc >= k || r > k) av = 0.0;
                            else if (r == k) av = cv[nl];           // bordered row: y_T
                            else if (r == cc) av = 1.0 + lam;       // exp(0) + lambda
                            else if (r < cc) av = 0.0;              // upper triangle: unused
                            else {
                                const double dx = rx[ml] - cx[nl], dy = ry[ml] - cy[nl];
                                av = exp(sqrt(dx * dx + dy * dy) * ninv);
                            }
                            Cs[nl * AS + ml] = av - acc[i][j][e];
                        }
                __syncthreads();

                if (rt == 0) {
                    // Fused unblocked Cholesky of C[0:jw,0:jw] and inverse of its factor.
                    for (int e = tid; e < BT_DBL; e += NT) Bt[e] = 0.0;
                    if (tid == 0) s_fail = 0;
                    __syncthreads();
                    for (int i = tid; i < jw; i += NT) Bt[i * BS + i] = 1.0;
                    __syncthreads();
                    for (int q = 0; q < jw; ++q) {
                        const double d = Cs[q * AS + q];
                        if (!(d > 0.0)) {  // not positive definite (R12); uniform decision
                            if (tid == 0) s_fail = 1;
                            break;
                        }
                        const double sd = sqrt(d);
                        const double inv = 1.0 / sd;
                        if (tid == 0) dg[q] = sd;
                        for (int r = q + 1 + tid; r < jw; r += NT) Cs[q * AS + r] *= inv;
                        for (int i = tid; i <= q; i += NT) Bt[i * BS + q] *= inv;
                        __syncthreads();
                        const int w = jw - q - 1;
                        for (int e = tid; e < w * w; e += NT) {
                            const int cc = q + 1 + e / w, r = q + 1 + e % w;
                            if (r >= cc) Cs[cc * AS + r] -= Cs[q * AS + r] * Cs[q * AS + cc];
                        }
                        for (int e = tid; e < w * (q + 1); e += NT) {
                            const int n = q + 1 + e % w, i = e / w;
                            Bt[i * BS + n] -= Cs[q * AS + n] * Bt[i * BS + q];
                        }
                        __syncthreads();
                    }
                    __syncthreads();
                    if (s_fail) {
                        failed = true;
                        break;
                    }
                }

                // X = C . Linv^T (triangular solve against L_jj^T as a GEMM)
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
                mma_tile<NB / 4>(acc, Cs, AS, Bt, BS, wm, wn, g, t);

#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int ml = wm * 32 + i * 8 + g;
                            const int nl = wn * 32 + j * 8 + 2 * t + e;
                            const int r = r0 + ml;
                            if (nl >= jw || r > k) continue;
                            double val;
                            if (rt == 0 && ml < jw) {
                                if (ml < nl) continue;
                                val = ml == nl ? dg[nl] : Cs[nl * AS + ml];
                            } else {
                                val = acc[i][j][e];
                            }
                            L[(size_t)(j0 + nl) * ld + r] = val;
                        }
                __threadfence_block();
                __syncthreads();
            }
        }

        if (failed) {
            if (tid == 0) {
                a.subset_loss[(int64_t)s * a.C + c] = __longlong_as_double(0x7ff8000000000000ll);
                a.fail[(int64_t)s * a.C + c] = 1;
            }
            continue;
        }

        // ---------------- backward substitution L^T alpha = z ----------------
        double *alpha = stage;  // k doubles (k <= STAGE_DBL)
        double *LJ = Bt;        // NB x LJS
        double *tvec = rx;      // NB
        for (int jb = nblk - 1; jb >= 0; --jb) {
            const int j0 = jb * NB;
            const int jw = min(NB, k - j0);
            const int rs = j0 + jw;
            for (int cl = warp; cl < jw; cl += NT / 32) {
                const double *col = L + (size_t)(j0 + cl) * ld;
                double sum = 0.0;
                for (int r = rs + lane; r < k; r += 32) sum += __ldcg(col + r) * alpha[r];
                sum = warp_sum(sum);
                if (lane == 0) tvec[cl] = __ldcg(col + k) - sum;  // z_c - L[c+1:, c] . alpha
            }
            for (int e = tid; e < jw * jw; e += NT) {
                const int cc = e / jw, rr = e % jw;  // column cc, row rr of the block
                if (rr >= cc) LJ[rr * LJS + cc] = __ldcg(L + (size_t)(j0 + cc) * ld + j0 + rr);
            }
            __syncthreads();
            if (warp == 0) {
                double t0 = lane < jw ? tvec[lane] : 0.0;
                double t1 = lane + 32 < jw ? tvec[lane + 32] : 0.0;
                for (int cc = jw - 1; cc >= 0; --cc) {
                    const double tc = __shfl_sync(0xffffffffu, cc < 32 ? t0 : t1, cc & 31);
                    const double al = tc / LJ[cc * LJS + cc];
                    if (lane < cc) t0 -= LJ[cc * LJS + lane] * al;
                    if (lane + 32 < cc) t1 -= LJ[cc * LJS + lane + 32] * al;
                    if (lane == 0) alpha[j0 + cc] = al;
                }
            }
            __syncthreads();
        }

        // ---------------- prediction and squared error (Eq.3, Eq.4) ----------------
        const double *vx = a.vx + voff, *vy = a.vy + voff, *vv = a.vv + voff;
        double part = 0.0;
        for (int v = warp; v < m; v += NT / 32) {
            const double px = __ldg(vx + v), py = __ldg(vy + v);
            double sum = 0.0;
            for (int j = lane; j < k; j += 32) {
                const double dx = px - __ldg(tx + j), dy = py - __ldg(ty + j);
                sum += exp(sqrt(dx * dx + dy * dy) * ninv) * alpha[j];
            }
            sum = warp_sum(sum);
            const double e = sum - __ldg(vv + v);
            part += e * e;
        }
        if (lane == 0) red[warp] = part;
        __syncthreads();
        if (tid == 0) {
            double l = 0.0;
            for (int w = 0; w < NT / 32; ++w) l += red[w];
            a.subset_loss[(int64_t)s * a.C + c] = l;
            a.fail[(int64_t)s * a.C + c] = 0;
        }
    }
}

// loss[c] = sum_s subset_loss[s, c] in ascending s (Alg.1 line 9); status[c] = the
// smallest failing subset or -1.  One thread per config: a fixed, deterministic order.
__global__ void reduce_kernel(const double *subset_loss, const uint8_t *fail, int64_t N, int32_t C,
                              double *loss, int32_t *status) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    double acc = 0.0;
    int64_t st = -1;
    for (int64_t s = 0; s < N; ++s) {
        if (fail[s * C + c]) {
            if (st < 0) st = s;
        } else {
            acc += subset_loss[s * C + c];
        }
    }
    loss[c] = st >= 0 ? __longlong_as_double(0x7ff8000000000000ll) : acc;
    status[c] = (int32_t)st;
}

}  // namespace

size_t cv_kernel_smem_bytes() { return SMEM_BYTES; }
int cv_kernel_max_k() { return STAGE_DBL; }

cudaError_t cv_kernel_occupancy(int *blocks_per_sm) {
    cudaError_t e = cudaFuncSetAttribute(cv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)SMEM_BYTES);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, cv_kernel, NT, SMEM_BYTES);
}

cudaError_t launch_cv_kernel(const CvArgs &a, int grid, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(cv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)SMEM_BYTES);
    if (e != cudaSuccess) return e;
    cv_kernel<<<grid, NT, SMEM_BYTES, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_reduce(const double *subset_loss, const uint8_t *fail, int64_t N, int32_t C,
                          double *loss, int32_t *status, cudaStream_t st) {
    reduce_kernel<<<(C + 127) / 128, 128, 0, st>>>(subset_loss, fail, N, C, loss, status);
    return cudaGetLastError();
}

}  // namespace pgpcv
