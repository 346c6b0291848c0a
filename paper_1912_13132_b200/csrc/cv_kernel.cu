// cv_kernel.cu -- the hot path of parallel cross-validation on B200 (sm_100a), FP64.
//
// Persistent CTAs (two per SM) pull (subset s, config c) work items in LPT order and, for
// each, evaluate the subset's local SSPE z_i of Alg.1 line 7 exactly as
// Eq.3/Eq.4 define it:
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
// Data layout (per resident CTA, in HBM): L has k+1 rows (rows 0..k-1 the Cholesky factor,
// row k the bordered z; GLS adds p covariate rows) and k columns, stored in column groups
// of KC = 16: group q holds rows 16q..ld-1 (ld = roundup(k+1, 16); the packed lower
// triangle) with each row's 16 values contiguous (128 B) and XOR-swizzled by the row,
// L(r, c) at (gbase(q) + r)*16 + ((c & 15) ^ 4(r & 3)), q = c >> 4.
// An operand chunk (MT or NB consecutive rows of one column group) is then one
// contiguous 16 KB / 8 KB block: one bulk copy, and conflict-free DMMA fragment loads
// from the unpadded SMEM image.
//
// Left-looking step for block column j (width NB = 64, columns j0..j0+jw-1), for every
// row tile of MT = 128 rows r0.. (rows j0..k):
//   acc    = -A[r0:r0+MT, j0:j0+NB]                         -- generated in registers while
//            the tile's first operand chunks are in flight
//   acc   += L[r0:r0+MT, 0:j0] . L[j0:j0+NB, 0:j0]^T       -- FP64 DMMA (mma.m8n8k4),
//            operands streamed HBM/L2 -> SMEM by 1-D bulk copies (cp.async.bulk, one
//            16 KB + one 8 KB copy per chunk of KC = 16 columns) issued by one thread,
//            3 SMEM stages tracked by full/empty mbarriers (no CTA-wide barrier in the
//            loop) plus L2 prefetches (cp.async.bulk.prefetch.L2) PFD chunks further ahead
//   C      = -acc
//   tile 0 : L_jj = chol(C[0:jw, 0:jw]) and Linv = L_jj^{-1} in SMEM: 8-column panels
//            factored by warp 0 (rsqrt pivots, register shuffles), Linv rows finished
//            per panel, the previous panel's far trailing update by warps 1-7 meanwhile
//            (look-ahead); 16 CTA barriers per block.  Linv is also kept in the slot.
//   X      = C . Linv^T                                      -- FP64 DMMA; the A operand
//            comes straight from the accumulator registers via warp shuffles
//   L[r0:, j0:j0+jw] = X   (tile 0: its first jw rows are L_jj itself)
// After the last block column: alpha by blocked back-substitution (warp dot products
// below each diagonal block + the block's stored inverse), then the prediction.
//
// Each warp owns 16 full rows of a tile (8 warps x 16 = 128), so the TRSM needs no
// cross-warp exchange; a warp whose rows all lie in a tile's padding skips the update.
// ~111 KB of SMEM and <= 128 registers per thread let two CTAs share an SM, so one CTA's
// barriers, epilogue, diagonal factorization and back-substitution overlap the other's
// DMMA stream.  The FP64 ALU work outside the update (the covariance's exp/sqrt, the
// pivots) shares the FP64 pipe with DMMA, so it is kept short: a table-driven exp for
// x <= 0 and branch-free generation.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdint>

#include "pgpcv_internal.h"
#include "pgpcv_device.cuh"

namespace pgpcv {
namespace {

constexpr int KC = 16;       // = the column-group width of the factor layout
#ifndef PGPCV_PFD
#define PGPCV_PFD 4
#endif
constexpr int PFD = PGPCV_PFD;  // L2 prefetch distance beyond the SMEM stages (chunks)
// Where thread 0 refills the operand ring within a chunk: at its start (0) or after that many
// of its warp's four k-slices.  The refill waits until every warp released the stage's previous
// use, so the issuing warp starts each chunk last; a quarter chunk later the others have
// usually released it already.  Same-box A/B (profiles/r02d_ab_issue_at.json, reproduced in
// r02d_ab_poll.json): large kernel (c5) +1.0 % at 1, +0.7 % at 2; small kernel (c3, c4) -0.6 % / -1.3 %: its short tiles need
// the earliest issue.
#ifndef PGPCV_ISSUE_AT_LARGE
#define PGPCV_ISSUE_AT_LARGE 1
#endif
#ifndef PGPCV_ISSUE_AT_SMALL
#define PGPCV_ISSUE_AT_SMALL 0
#endif
// 1 = non-blocking refills: thread 0 polls the stage's empty barrier at every k-slice and
// issues as soon as it is free (up to STAGES - 1 chunks ahead); it blocks only for the chunk
// it is about to consume.  Measured slower on the same box (large kernel, c5: -2.3 % against
// ISSUE_AT 0, -3.2 % against ISSUE_AT 1; small kernel, c3: -14 %, c4: -6.5 %;
// profiles/r02d_ab_poll.json): the polls and their warp re-convergence sit in warp 0's DMMA
// stream.  Off.
#ifndef PGPCV_POLL_LARGE
#define PGPCV_POLL_LARGE 0
#endif
#ifndef PGPCV_POLL_SMALL
#define PGPCV_POLL_SMALL 0
#endif
#ifndef PGPCV_PFD_SMALL  // the same for the small-subset kernel (Geo<64, 32, ...>)
#define PGPCV_PFD_SMALL PGPCV_PFD
#endif

// Kernel geometry.  Two instantiations:
//   Geo<128, 64, 2>: the large-subset kernel -- 8 warps, row tiles of MT = 128, block
//     columns of NB = 64, two CTAs per SM (111 KB SMEM each);
//   Geo<64, 32, 4>:  the small-subset kernel -- 4 warps, MT = 64, NB = 32, four CTAs per SM
//     (47 KB each): at k of a few hundred the per-item critical path (the diagonal blocks'
//     pivot chain, the TRSM, the back-substitution) dominates, and twice the items in
//     flight per SM hide it; its operands stream at 5.3 instead of 10.7 flop/B.
// Each warp owns 16 full rows x NB columns of a row tile.
template <int MT_, int NB_, int MINB_, bool BORDER_, int STAGES_ = 3, bool SIG_ = false, bool WS_ = false>
struct Geo {
    static constexpr int MT = MT_, NB = NB_, MINB = MINB_;
    static constexpr bool BORDER = BORDER_;  // bordered prediction compiled in
    static constexpr int PFD = MT_ == 64 ? PGPCV_PFD_SMALL : PGPCV_PFD;  // L2 prefetch distance
    static constexpr int ISSUE_AT = MT_ == 64 ? PGPCV_ISSUE_AT_SMALL : PGPCV_ISSUE_AT_LARGE;  // refill position
    static constexpr bool POLL = !WS_ && (MT_ == 64 ? PGPCV_POLL_SMALL : PGPCV_POLL_LARGE);  // non-blocking refills
    static constexpr bool SIG = SIG_;        // covariance entries read from the per-range blocks
    // Warp-specialised CTA (WS): two consumer groups of NWARP warps, each an independent
    // "virtual CTA" with its own item, SMEM and named barrier, plus a producer warpgroup whose
    // warp g issues group g's operand chunks (setmaxnreg moves its registers to the consumers)
    static constexpr bool WS = WS_;
    static constexpr int GROUPS = WS ? 2 : 1;
    static constexpr int NWARP = MT / 16, NT = 32 * NWARP;
    static constexpr int THREADS = GROUPS * NT + (WS ? 128 : 0);  // block size at launch
    static constexpr int STAGES = STAGES_;
    static constexpr int BS = NB + 4;   // Linv^T row stride: 2 BS == 8 (mod 32) words, conflict-free fragments
    static constexpr int LJS = NB + 1;  // row stride of the diagonal block in SMEM
    static constexpr int A_STAGE = MT * KC;
    static constexpr int B_STAGE = NB * KC;
    static constexpr int STAGE_DBL = STAGES * (A_STAGE + B_STAGE);
    static constexpr int BT_DBL = NB * BS;                  // Linv^T tile
    static constexpr int COL_DBL = 3 * NB;                  // block-column x, y, value
    static constexpr int MISC_DBL = 2 * NB + NWARP + 64;    // pivots, warp partials, exp table
    static constexpr size_t SMEM_BYTES = sizeof(double) * (STAGE_DBL + BT_DBL + COL_DBL + MISC_DBL);
    static constexpr unsigned STAGE_BYTES = (unsigned)(KC * (MT + NB) * sizeof(double));
    static_assert(2 * NB * LJS <= STAGE_DBL, "diagonal block and its inverse must fit in the stage buffers");
    static_assert(NB * LJS <= BT_DBL, "back-substitution block must fit in the Linv buffer");
    static constexpr size_t CTA_SMEM = GROUPS * SMEM_BYTES;  // dynamic SMEM of one CTA
    static_assert(CTA_SMEM * MINB <= 232448 - MINB * 1024, "MINB CTAs per SM");
    static_assert((BS * 2) % 32 == 8, "fragment-load stride of Linv^T");
    static_assert(MT == 16 * NWARP && (NB == 64 || NB == 32) && MT >= NB, "warp tile 16 x NB");
};
using GeoLarge = Geo<kMT, kNB, 2, false>;
// the large kernel as one warp-specialised CTA per SM (two consumer groups + producers)
using GeoLargeWS = Geo<kMT, kNB, 1, false, 3, false, true>;
// setmaxnreg (CTA pool: 640 threads launch at 96 registers): the producer warpgroup gives up
// 128 x (96 - 32), the four consumer warpgroups take 512 x (112 - 96) of it
constexpr int kWsConsumerRegs = 112;
constexpr int kWsProducerRegs = 32;
// (5 or 6 CTAs per SM with a 2-stage ring were measured slower: r02_ab_small_occupancy.json)
#ifndef PGPCV_SMALL_MINB
#define PGPCV_SMALL_MINB 4
#endif
#ifndef PGPCV_SMALL_STAGES
#define PGPCV_SMALL_STAGES 3
#endif
using GeoSmall = Geo<kMTSmall, kNBSmall, PGPCV_SMALL_MINB, true, PGPCV_SMALL_STAGES>;
// the same small kernel reading the covariance from sigma_kernel's per-range blocks (a
// separate instantiation: the generating variant keeps its register allocation and schedule)
using GeoSmallSig = Geo<kMTSmall, kNBSmall, PGPCV_SMALL_MINB, true, PGPCV_SMALL_STAGES, true>;

// ---------------------------------------------------------------- mbarrier / bulk copy
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    unsigned done = 0;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ bool mbar_test(uint64_t *bar, unsigned parity) {  // non-blocking
    unsigned done;
    asm volatile(
        "{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return done != 0;
}
// 1-D bulk copy global -> shared (async proxy), completion counted on `bar` in bytes.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void add_release_u32(unsigned *p, unsigned v) {
    asm volatile("red.release.cta.shared::cta.add.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
// spin (with back-off) until the shared counter reaches `target` (WS hand-offs)
__device__ __forceinline__ void wait_count(const unsigned *p, unsigned target) {
    while ((int)(ld_acquire_u32(p) - target) < 0) __nanosleep(32);
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.global;\n fence.proxy.async.shared::cta;" ::: "memory");
}


// Diagnostic build only (-DPGPCV_PHASE_PROFILE, probes/p2_phases.py): thread 0 of every CTA
// attributes its clock64() time to the phases below; the API prints the sums per launch.
#ifdef PGPCV_PHASE_PROFILE
#ifdef PGPCV_TIMELINE
// Timeline (probes/p3_timeline.py): thread 0 logs the SM clock each time its CTA switches
// between the update (phases 3-4) and anything else; word 0 of a CTA's log is its SM id.
constexpr int kTimelineLen = 1 << 15;
#define TL_LOG(i, t0)                                                                        \
    do {                                                                                     \
        const int st_ = ((i) == 3 || (i) == 4) ? 1 : 0;                                      \
        if (st_ != tl_state && a.tl && tl_n < kTimelineLen - 2) {                            \
            a.tl[(size_t)slot * kTimelineLen + 2 + tl_n++] = ((unsigned long long)(t0) << 1) | st_; \
            tl_state = st_;                                                                  \
        }                                                                                    \
    } while (0)
#define TL_DECL int tl_state = -1, tl_n = 0;
#else
#define TL_LOG(i, t0) \
    do {              \
    } while (0)
#define TL_DECL
#endif
#define PH_DECL long long ph_t = clock64(); TL_DECL
#define PH(i)                                   \
    do {                                        \
        if (tid == 0) {                         \
            const long long t_ = clock64();     \
            s_ph[i] += (unsigned long long)(t_ - ph_t); \
            TL_LOG(i, ph_t);                    \
            ph_t = t_;                          \
        }                                       \
    } while (0)
#else
#define PH_DECL
#define PH(i) \
    do {      \
    } while (0)
#endif
// 0 item fetch/setup, 1 block-column setup, 2 A generation, 3 GEMM issue/compute,
// 4 GEMM operand wait, 5 barrier after tile 0's GEMM, 6 diagonal factorization + inverse,
// 7 L_jj store + barrier, 8 TRSM + stores, 9 end-of-column fence + barrier,
// 10 back-substitution, 11 prediction + outputs; within 6: 12 diagonal setup, 13 panel
// factorization (warp 0), 14 trailing updates and their barriers
constexpr int kPhases = 15;

// Packed lower-triangular storage: column group q (columns 16q..16q+15) is only ever read or
// written at rows >= 16q, so it stores rows 16q..ld-1; groups follow each other.  Row r of
// group q starts at (gbase(q) + r) * 16 with gbase(q) = sum_{q'<q} (ld - 16q') - 16q.
__host__ __device__ __forceinline__ int64_t gbase(int64_t ld, int64_t q) { return q * ld - 8 * q * (q + 1); }
// doubles of a packed factor with G column groups
__host__ __device__ __forceinline__ int64_t factor_doubles(int64_t ld, int64_t G) {
    return (G * ld - 8 * G * (G - 1)) * KC;
}
// Element (r, c) of the factor in the column-group tiled, row-swizzled layout.
__device__ __forceinline__ size_t lidx(int64_t ld, int r, int c) {
    return (size_t)(gbase(ld, c >> 4) + r) * KC + ((c & 15) ^ ((r & 3) << 2));
}
// Start of the contiguous chunk rows r.. of column group q.
__device__ __forceinline__ const double *lchunk(const double *L, int64_t ld, int q, int r) {
    return L + (size_t)(gbase(ld, q) + r) * KC;
}

// Operand chunk n of the running sequence (stage n % STAGES, use n / STAGES): one thread
// waits until every warp released the stage's previous use, then issues two bulk copies:
// rows r0..r0+MT-1 (A) and j0..j0+NB-1 (B) of column group kk/16.  Rows past the matrix
// are copied as whatever the workspace holds; they only reach discarded outputs (see the
// masking of acc after the update).  Chunk n + PFD is prefetched into L2.
// (block = false: only if the stage is free already; returns whether the chunk was issued)
template <class G>
__device__ __forceinline__ bool issue_chunk(uint32_t n, double *stage, uint64_t *full, uint64_t *empty,
                                            const double *L, int64_t ld, int r0, int j0, int kk,
                                            bool block = true) {
    const int sidx = n % G::STAGES;
    const uint32_t use = n / G::STAGES;
    if (use > 0) {
        if (block) mbar_wait(&empty[sidx], (use - 1) & 1);
        else if (!mbar_test(&empty[sidx], (use - 1) & 1)) return false;
    }
    double *sb = stage + sidx * (G::A_STAGE + G::B_STAGE);
    mbar_expect_tx(&full[sidx], G::STAGE_BYTES);
    bulk_g2s(sb, lchunk(L, ld, kk / KC, r0), G::MT * KC * sizeof(double), &full[sidx]);
    bulk_g2s(sb + G::A_STAGE, lchunk(L, ld, kk / KC, j0), G::NB * KC * sizeof(double), &full[sidx]);
    return true;
}
template <class G>
__device__ __forceinline__ void prefetch_chunk(const double *L, int64_t ld, int r0, int j0, int kk) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lchunk(L, ld, kk / KC, r0)),
                 "r"((unsigned)(G::MT * KC * sizeof(double)))
                 : "memory");
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lchunk(L, ld, kk / KC, j0)),
                 "r"((unsigned)(G::NB * KC * sizeof(double)))
                 : "memory");
}
// Refill protocol: 0 = thread 0 issues chunk n + STAGES - 1 at the start of chunk n after
// waiting for every release (round 1); 1 = the last warp to release a stage refills it, the
// tile prologue issuing all STAGES chunks; 2 = as 1, but the prologue issues STAGES - 1 and
// thread 0 the last one at the tile's first chunk.
#ifndef PGPCV_LAST_REFILLS
#define PGPCV_LAST_REFILLS 0
#endif
// Consumer-side fence.proxy.async before a stage is released: 0 (default since round 2) --
// the release's mbarrier arrive (release semantics) and the producer's wait (acquire) order
// the warps' generic-proxy fragment reads before the async-proxy refill of the stage, a
// write-after-read the bulk copy may follow without a proxy fence (the cross-proxy fences
// stay where generic WRITES to stage memory -- the diagonal block, alpha, z -- precede a
// refill).  Same-box A/B: c5 +0.4 %, c3/c4 +0.2 %; 40 stress repetitions of the c2 grid on
// both kernel variants and the whole GPU suite bit-clean (profiles/r02_ab_loop_fence.json).
// 1 restores the round-1 fence.
#ifndef PGPCV_LOOP_FENCE
#define PGPCV_LOOP_FENCE 0
#endif
// Column of the i-th operand chunk of a tile: ascending on even row tiles, descending on
// odd ones (a boustrophedon over the k-chunks), so a tile starts with the B-panel chunks
// the previous tile of the same block column read last -- still in L2.
#ifndef PGPCV_PAIR_STORE  // TRSM epilogue: 16-B stores of column pairs (0: 8-B stores, round 1)
#define PGPCV_PAIR_STORE 1
#endif
#ifndef PGPCV_SNAKE
#define PGPCV_SNAKE 1
#endif
// 1 = the operand ring runs on across row tiles (see the update loop).  Measured slower on
// the same box (c3 -3.9 %, c4 -0.7 %, c5 -0.4 %; profiles/r02d_ab_runahead.json): thread 0
// then waits for every warp's release in the last chunks of a tile too, where it otherwise
// catches up with the other warps.  Off.
#ifndef PGPCV_RUNAHEAD
#define PGPCV_RUNAHEAD 0
#endif
// Diagonal panel (warp 0): 1 = the pivot chain through a reciprocal estimate with the
// correction folded into the multiplier, and Linv rows pre-scaled (shorter FP64 chains);
// 0 = the round-1 chain through rsqrt_nb.
#ifndef PGPCV_PIVOT_RCP
#define PGPCV_PIVOT_RCP 0
#endif
__device__ __forceinline__ int chunk_col(int i, int nk, bool rev) { return (PGPCV_SNAKE && rev ? nk - 1 - i : i) * KC; }
// Tile prologue: SMEM chunks 0..STAGES-2 and L2 prefetches of the next PFD chunks.
// (issued = true: the previous tile's update loop already issued the SMEM chunks, PGPCV_RUNAHEAD)
// Returns the number of SMEM chunks issued (POLL: only those whose stage was free).
template <class G>
__device__ __forceinline__ int tile_prologue(uint32_t pc, int nk, double *stage, uint64_t *full,
                                             uint64_t *empty, const double *L, int64_t ld, int r0,
                                             int j0, bool rev, bool issued = false) {
    fence_proxy_async();
    constexpr int PRO = PGPCV_LAST_REFILLS == 1 ? G::STAGES : G::STAGES - 1;  // chunks in flight at tile start
    int ni = 0;
    for (int i = 0; i < min(PRO, nk) && !issued; ++i) {
        if (!issue_chunk<G>(pc + i, stage, full, empty, L, ld, r0, j0, chunk_col(i, nk, rev), !G::POLL)) break;
        ++ni;
    }
    for (int i = PRO; i < min(PRO + G::PFD, nk); ++i)
        prefetch_chunk<G>(L, ld, r0, j0, chunk_col(i, nk, rev));
    return ni;
}

template <class G>
__device__ void ws_producer(const CvArgs &a, double *stage, uint64_t *full, uint64_t *empty, const double *L,
                           const unsigned *go, unsigned *ack, const int *s_item, const int *s_fail);

template <class G>
__global__ void __launch_bounds__(G::THREADS, G::MINB) cv_kernel(CvArgs a) {
    constexpr int MT = G::MT, NB = G::NB, NT = G::NT, NWARP = G::NWARP, STAGES = G::STAGES;
    constexpr int BS = G::BS, LJS = G::LJS, A_STAGE = G::A_STAGE, B_STAGE = G::B_STAGE;
    constexpr int STAGE_DBL = G::STAGE_DBL, BT_DBL = G::BT_DBL;
    constexpr int NJ = NB / 8;  // 8-column fragments per warp row block
    extern __shared__ __align__(128) double smem_all[];
    // WS: warps 0..2 NWARP-1 are the consumers of groups 0 and 1, warp 2 NWARP + g the
    // producer of group g (g < 2; the warpgroup's other two warps only donate registers)
    const int wid = threadIdx.x >> 5;
    const bool producer = G::WS && wid >= G::GROUPS * NWARP;
    const int grp = G::WS ? (producer ? wid - G::GROUPS * NWARP : wid / NWARP) : 0;
    const int gs = grp < G::GROUPS ? grp : G::GROUPS - 1;  // this thread's group state
    const int slot = G::WS ? blockIdx.x * G::GROUPS + gs : blockIdx.x;  // factor slot / output row
    double *smem = smem_all + (size_t)gs * (G::SMEM_BYTES / sizeof(double));
    double *stage = smem;
    double *LJ = smem;                  // diagonal block [r][c], aliases the stages
    double *Bt = smem + STAGE_DBL;      // Bt[q*BS + n] = Linv[n][q]
    double *cx = Bt + BT_DBL;           // block-column coordinates and values
    double *cy = cx + NB;
    double *cv = cy + NB;
    double *dg = cv + NB;               // sqrt pivots of the diagonal block
    double *red = dg + 2 * NB;          // per-warp partial sums
    double *etab = red + NWARP;         // 2^(j/64), j = 0..63 (exp_neg)
    __shared__ __align__(8) uint64_t full_a[G::GROUPS][STAGES];
    __shared__ __align__(8) uint64_t empty_a[G::GROUPS][STAGES];
    __shared__ int s_item_a[G::GROUPS];
    __shared__ int s_fail_a[G::GROUPS];
    __shared__ int s_rank_a[G::GROUPS];  // arrival order of this CTA on its SM (sched 1)
    __shared__ unsigned rel_a[G::GROUPS][STAGES];  // releases of each stage's current use (PGPCV_LAST_REFILLS)
    __shared__ unsigned go_a[G::GROUPS], ack_a[G::GROUPS];  // WS hand-offs (consumer -> producer, back)
    uint64_t *full = full_a[gs], *empty = empty_a[gs];
    int &s_item = s_item_a[gs];
    int &s_fail = s_fail_a[gs];
    int &s_rank = s_rank_a[gs];
    unsigned *rel = rel_a[gs];
    unsigned *go = &go_a[gs], *ack = &ack_a[gs];
#ifdef PGPCV_PHASE_PROFILE
    __shared__ unsigned long long s_ph_a[G::GROUPS][kPhases];
    if (threadIdx.x < G::GROUPS * kPhases) (&s_ph_a[0][0])[threadIdx.x] = 0;
    unsigned long long *s_ph = s_ph_a[gs];
#endif

    const int tid = G::WS ? (int)threadIdx.x - gs * NT : (int)threadIdx.x;  // thread in the group
    const int lane = threadIdx.x & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    double *L = a.work + (size_t)slot * a.slot_stride;
    // barrier of this thread's group: the CTA (or, WS, the group's named barrier)
    auto gsync = [&]() {
        if constexpr (G::WS)
            asm volatile("bar.sync %0, %1;" ::"r"(gs + 1), "n"(NT) : "memory");
        else
            __syncthreads();
    };

    if (!producer && tid < EXP_TAB) etab[tid] = kExp2Tab[tid];
    if (!producer && tid == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NWARP);
            rel[i] = 0;
        }
        *go = 0;
        *ack = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        s_rank = a.sched == 1 && !G::WS ? (int)(atomicAdd(a.counter + 1 + (smid % kMaxSms), 1ull) & 1ull) : 0;
    }
    __syncthreads();  // the whole CTA, once
    if constexpr (G::WS) {
        if (producer) {
            asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kWsProducerRegs) : "memory");
            if (grp < G::GROUPS && lane == 0) ws_producer<G>(a, stage, full, empty, L, go, ack, &s_item, &s_fail);
            return;
        }
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kWsConsumerRegs) : "memory");
    }
    uint32_t pc = 0;  // operand chunks consumed so far (identical in every thread)
    uint32_t issued = 0;  // POLL, thread 0: operand chunks issued so far
    unsigned n_claims = 0;  // WS: items this group claimed (thread 0)
    PH_DECL

    for (;;) {
        if (tid == 0) {
            // WS: the producer has issued every chunk of the previous item (so it has read
            // s_item before it is overwritten here)
            if constexpr (G::WS) wait_count(ack, n_claims);
            // Claim the next item: from the front of the LPT list, or (sched 1, the SM's
            // second CTA) from the back, so the two CTAs sharing an SM work on subsets of
            // different sizes and their non-GEMM phases do not fall into step.  The sum of
            // both claim counts orders the claims: exactly n_items succeed, none twice.
            const bool back = a.sched == 1 && s_rank == 1;
            const unsigned long long old = atomicAdd(a.counter, back ? (1ull << 32) : 1ull);
            const long long f = (long long)(old & 0xffffffffull), b = (long long)(old >> 32);
            s_item = f + b < a.n_items ? (int)(back ? a.n_items - 1 - b : f) : a.n_items;
            if constexpr (G::WS) {  // hand-off 1: the item (or the end) to the producer
                ++n_claims;
                add_release_u32(go, 1);
            }
        }
        gsync();
        const int item = s_item;
        gsync();
        if (item >= a.n_items) {
#ifdef PGPCV_PHASE_PROFILE
            PH(0);
            if (tid < kPhases && a.prof) a.prof[slot * kPhases + tid] = s_ph[tid];
#ifdef PGPCV_TIMELINE
            if (tid == 0 && a.tl) {
                unsigned smid;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                a.tl[(size_t)slot * kTimelineLen] = smid;
                a.tl[(size_t)slot * kTimelineLen + 1] = (unsigned long long)tl_n;
            }
#endif
#endif
            break;
        }
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
        const int np = (a.flags & kCvGls) ? a.p : 0;  // covariate rows bordered below y (f4)
        // Bordered prediction (border_pred): the m targets' cross-covariance rows b_v are
        // bordered below y, so the factorization's forward sweep leaves w_v = L^{-1} b_v in
        // row k+1+v and yhat_v = b_v^T (L L^T)^{-1} y = w_v . z -- no back-substitution.
        // Per item: bordering costs m k^2 DMMA flops (3m/k of the factorization); it replaces
        // the back-substitution only while m <= k / 20 (c3, c4; c2's m/k ~ 0.06 measured
        // 1.3 % slower bordered).  border_pred 2 borders every item (tests).
        const int nbt = G::BORDER ? (int)border_rows(a.flags, a.border_pred, k, m) : 0;
        const int kb = k + np + nbt;                    // last bordered row
        const double *vxi = a.vx + voff, *vyi = a.vy + voff;
        const int64_t ld = factor_ld(kb);
        const int nblk = (k + NB - 1) / NB;
        // This subset's covariance for this range, generated once per call (sigma_kernel),
        // when the call reuses it (small kernel only); else nullptr: generate per item.
        const double *sg = nullptr;
        if constexpr (G::SIG) sg = a.sig + (size_t)a.sig_range[c] * a.sig_stride + a.sig_off[s];
        const int64_t sld = sigma_ld(k, nbt);
        // L2 prefetch of the per-range block's rows r0..r0+MT-1 of the block column's groups
        // (issued one row tile ahead, so the tile's entry loads hit L2)
        auto sig_prefetch = [&](int r0p, int j0p) {
            if constexpr (G::SIG) {
                const int rows = min(MT, (int)(k + nbt + 1) - r0p);
                if (rows <= 0) return;
                for (int q = j0p / KC; q < (j0p + NB) / KC && q * KC < k; ++q)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(sg + (size_t)(gbase(sld, q) + r0p) * KC),
                                 "r"((unsigned)(rows * KC * sizeof(double)))
                                 : "memory");
            }
        };
        const int64_t oi = (int64_t)s * a.out_C + (a.out_C > 1 ? c : 0);  // output entry
        // slot scratch after the packed factor: alpha (k, when not in SMEM), then the
        // inverse of every diagonal block (nblk x 64 x 64, row-major) for the solves
        double *linvG = L + factor_doubles(ld, (k + KC - 1) / KC) + ((k + 31) / 32) * 32;
        bool failed = false;
        double logdet = 0.0;  // sum_i log L_ii (warp 0, kCvNll)

        // ---------------- blocked left-looking Cholesky with bordered y row ----------------
        for (int jb = 0; jb < nblk && !failed; ++jb) {
            const int j0 = jb * NB;
            const int jw = min(NB, k - j0);
            const int nrows = kb + 1 - j0;  // rows j0..kb (row k: bordered y, then covariates)
            const int ntiles = (nrows + MT - 1) / MT;
            const int nk = j0 / KC;        // operand chunks per tile
            for (int i = tid; i < NB; i += NT) {
                const int cc = j0 + i;
                const bool ok = cc < k;
                cx[i] = ok ? __ldg(tx + cc) : 0.0;
                cy[i] = ok ? __ldg(ty + cc) : 0.0;
                cv[i] = ok ? __ldg(tv + cc) : 0.0;
            }
            // The previous block column's factor stores (generic proxy, made GPU-visible
            // before the last barrier) are read next by bulk copies (async proxy); the
            // stage memory was last touched by generic accesses (LJ, alpha).
            PH(0);
            if (!G::WS && tid == 0) {  // (WS: the producer issues every chunk)
                issued = pc + tile_prologue<G>(pc, nk, stage, full, empty, L, ld, j0, j0, false);
                if (jb == 0) sig_prefetch(j0, j0);
            }
            __syncwarp();
            gsync();  // cx/cy/cv visible
            PH(1);
            for (int rt = 0; rt < ntiles; ++rt) {
                const int r0 = j0 + rt * MT;
                const int rbase = r0 + warp * 16;  // this warp's first row
                double acc[2][NJ][2];

                const bool live = rbase <= kb;  // this warp holds at least one row of the matrix
                // (Skipping the diagonal-block warps' upper fragments in tile 0 -- generation
                // and DMMAs -- was measured slower at every k: c3 -13 %, c4 -5 %, c5 +0.0 %;
                // profiles/r02_ab_diagskip.json.  Only whole padding warps skip.)

                // acc = -A[r0:r0+MT, j0:j0+NB] (Eq.3 second line), generated while
                // the first operand chunks of the tile are in flight.
                {
                    double rx[2], ry[2];
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        const int r = rbase + i * 8 + g;
                        const bool tgt = G::BORDER && nbt > 0 && r > k && r <= kb;  // bordered target row
                        rx[i] = r < k ? __ldg(tx + r) : (tgt ? __ldg(vxi + (r - k - 1)) : 0.0);
                        ry[i] = r < k ? __ldg(ty + r) : (tgt ? __ldg(vyi + (r - k - 1)) : 0.0);
                    }
                    // all 32 entries without branches (independent chains the scheduler can
                    // interleave); the special entries by selects.  (Generating the next
                    // tile's entries inside the update loop instead was measured 5 % slower:
                    // the exp chains then compete with the DMMA stream of the same warp.)
                    auto gen = [&](int i, int j, int e) {
                        const int r = rbase + i * 8 + g;
                        const int nl = j * 8 + 2 * t + e;
                        const int cc = j0 + nl;
                        double v = -cov_exp(rx[i] - cx[nl], ry[i] - cy[nl], ninv, etab);
                        v = r == cc ? -(1.0 + lam) : v;                 // exp(0) + lambda
                        v = r == k ? -cv[nl] : v;                       // bordered y_T
                        v = (cc >= k || r > kb || r < cc) ? 0.0 : v;    // pad / upper
                        acc[i][j][e] = v;
                    };
                    if constexpr (G::SIG) {
                      if (live) {
                        // the entries of Sigma_theta from the per-range block (16-B loads of
                        // the (2t, 2t+1) column pairs), then the same diagonal / y / padding
                        // rules as the generation: bit-identical to generating them here
#pragma unroll
                        for (int i = 0; i < 2; ++i) {
                            const int r = rbase + i * 8 + g;
                            const bool rok = r < k || (r > k && r <= k + nbt);
#pragma unroll
                            for (int j = 0; j < NJ; ++j) {
                                const int c0 = j0 + j * 8 + 2 * t;
                                double2 w = make_double2(0.0, 0.0);
                                if (rok && c0 < k) w = __ldg(reinterpret_cast<const double2 *>(sg + lidx(sld, r, c0)));
                                acc[i][j][0] = w.x;
                                acc[i][j][1] = w.y;
                            }
                        }
#pragma unroll
                        for (int i = 0; i < 2; ++i)
#pragma unroll
                            for (int j = 0; j < NJ; ++j)
#pragma unroll
                                for (int e = 0; e < 2; ++e) {
                                    const int r = rbase + i * 8 + g;
                                    const int nl = j * 8 + 2 * t + e;
                                    const int cc = j0 + nl;
                                    double v = -acc[i][j][e];
                                    v = r == cc ? -(1.0 + lam) : v;
                                    v = r == k ? -cv[nl] : v;
                                    v = (cc >= k || r > kb || r < cc) ? 0.0 : v;
                                    acc[i][j][e] = v;
                                }
                      } else {
#pragma unroll
                        for (int i = 0; i < 2; ++i)
#pragma unroll
                            for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
                      }
                    } else if (live) {
#pragma unroll
                        for (int i = 0; i < 2; ++i)
#pragma unroll
                            for (int j = 0; j < NJ; ++j)
#pragma unroll
                                for (int e = 0; e < 2; ++e) gen(i, j, e);
                    } else {  // a warp of the last tile's padding: nothing to generate
#pragma unroll
                        for (int i = 0; i < 2; ++i)
#pragma unroll
                            for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
                    }
                    if (np > 0) {  // bordered covariate rows (GLS, row f4)
#pragma unroll
                        for (int i = 0; i < 2; ++i)
#pragma unroll
                            for (int j = 0; j < NJ; ++j)
#pragma unroll
                                for (int e = 0; e < 2; ++e) {
                                    const int r = rbase + i * 8 + g;
                                    const int cc = j0 + j * 8 + 2 * t + e;
                                    if (r > k && r <= kb && cc < k)
                                        acc[i][j][e] = -__ldg(a.tX + (toff + cc) * np + (r - k - 1));
                                }
                    }
                }

                PH(2);
                // acc += L[r0:r0+MT, 0:j0] . L[j0:j0+NB, 0:j0]^T
                const int sw = (g & 3) << 2;  // fragment swizzle (row & 3 == g & 3)
                // Run-ahead: from row tile 1 on, the operand ring runs on into the next row
                // tile of the block column (its operands are earlier block columns, final
                // since the column's start), so the first chunks of tile rt + 1 are in flight
                // during the last chunks of tile rt instead of from its TRSM on.  Not from
                // tile 0: the diagonal block reuses the stage memory between the two.
                const bool run_next = PGPCV_RUNAHEAD && PGPCV_LAST_REFILLS == 0 && !G::WS && rt >= 1 &&
                                      rt + 1 < ntiles && nk >= STAGES - 1;
                for (int kc = 0; kc < nk; ++kc) {
                    const uint32_t n = pc + kc;
                    // (PGPCV_ISSUE_AT: thread 0 refills at the start of the chunk (0) or after
                    // that many of its warp's k-slices, when the other warps have more likely
                    // released the stage already)
                    auto refill = [&]() {
                      if (!G::WS && tid == 0 && (PGPCV_LAST_REFILLS != 1) && (PGPCV_LAST_REFILLS == 0 || kc == 0)) {
                        if (kc + STAGES - 1 < nk)
                            issue_chunk<G>(n + STAGES - 1, stage, full, empty, L, ld, r0, j0,
                                           chunk_col(kc + STAGES - 1, nk, rt & 1));
                        else if (run_next)
                            issue_chunk<G>(n + STAGES - 1, stage, full, empty, L, ld, r0 + MT, j0,
                                           chunk_col(kc + STAGES - 1 - nk, nk, (rt + 1) & 1));
                        // (running this L2 prefetch on into the next row tile's first chunks
                        // measured slower: c3 -4 %, c4 -2 %, c5 -0.3 %; r02_ab_xtile_prefetch.json)
                        if (kc + STAGES - 1 + G::PFD < nk)
                            prefetch_chunk<G>(L, ld, r0, j0, chunk_col(kc + STAGES - 1 + G::PFD, nk, rt & 1));
                      }
                    };
                    if constexpr (G::POLL) {
                        if (tid == 0) {
                            // the chunk about to be consumed (and any before it) must be in flight
                            while ((int)(issued - n) <= 0) {
                                issue_chunk<G>(issued, stage, full, empty, L, ld, r0, j0,
                                               chunk_col((int)(issued - pc), nk, rt & 1));
                                ++issued;
                            }
                            if (kc + STAGES - 1 + G::PFD < nk)
                                prefetch_chunk<G>(L, ld, r0, j0, chunk_col(kc + STAGES - 1 + G::PFD, nk, rt & 1));
                        }
                    } else if (G::ISSUE_AT == 0) {
                        refill();
                    }
                    PH(3);
                    mbar_wait(&full[n % STAGES], (n / STAGES) & 1);
                    PH(4);
                    __syncwarp();  // mma.sync.aligned needs the whole warp converged
                    const double *As = stage + (n % STAGES) * (A_STAGE + B_STAGE);
                    const double *ap = As + (warp * 16 + g) * KC + t;
                    const double *bp = As + A_STAGE + g * KC + t;
                    // A warp whose 16 rows all lie below the last bordered row (the padding
                    // of a tile that overhangs the matrix) issues no DMMA (warp-uniform).
                    if (live) {
#pragma unroll
                        for (int k4 = 0; k4 < KC / 4; ++k4) {
                            if constexpr (G::POLL) {  // (warp 0 is always live)
                                if (tid == 0 && (int)(issued - pc) <= min(kc + STAGES - 1, nk - 1) &&
                                    issue_chunk<G>(issued, stage, full, empty, L, ld, r0, j0,
                                                   chunk_col((int)(issued - pc), nk, rt & 1), false))
                                    ++issued;
                                __syncwarp();
                            } else if (G::ISSUE_AT > 0 && k4 == G::ISSUE_AT) {
                                refill();
                                __syncwarp();
                            }
                            const int o = (k4 << 2) ^ sw;
                            double af[2], bf[NJ];
                            af[0] = ap[o];
                            af[1] = ap[8 * KC + o];
#pragma unroll
                            for (int j = 0; j < NJ; ++j) bf[j] = bp[j * 8 * KC + o];
#pragma unroll
                            for (int j = 0; j < NJ; ++j)
#pragma unroll
                                for (int i = 0; i < 2; ++i) dmma(acc[i][j], af[i], bf[j]);
                        }
                    }
                    // Release the stage (PGPCV_LOOP_FENCE above: whether a proxy fence
                    // precedes the release).
#if PGPCV_LOOP_FENCE
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
                    __syncwarp();
                    if (lane == 0) {
                        mbar_arrive(&empty[n % STAGES]);
#if PGPCV_LAST_REFILLS
                        // The last warp to release the stage refills it with chunk n + STAGES
                        // at once: no fixed producer thread whose own warp lags behind the
                        // others (P6: 32.8 -> 34.6 TFLOP/s for the loop alone).
                        unsigned old;
                        asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                                     : "=r"(old) : "r"(smem_u32(&rel[n % STAGES])) : "memory");
                        if (old == NWARP - 1) {
                            rel[n % STAGES] = 0;
                            // (mode 2: chunk STAGES - 1 of a tile is issued by thread 0 at kc = 0,
                            // so the tile prologue never waits for the previous tile's last chunk)
                            if (kc + STAGES < nk)
                                issue_chunk<G>(n + STAGES, stage, full, empty, L, ld, r0, j0,
                                               chunk_col(kc + STAGES, nk, rt & 1));
                            if (kc + STAGES + G::PFD < nk)
                                prefetch_chunk<G>(L, ld, r0, j0, chunk_col(kc + STAGES + G::PFD, nk, rt & 1));
                        }
#endif
                    }
                }
                pc += nk;
                PH(3);
                // Columns past the matrix (last block column) came from rows of the
                // workspace beyond the factor: force C = 0 there (Linv^T is 0 there too).
#pragma unroll
                for (int j = 0; j < NJ; ++j)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        if (j0 + j * 8 + 2 * t + e >= k) acc[0][j][e] = acc[1][j][e] = 0.0;

                if (rt == 0) {
                    gsync();  // every warp is past the update: LJ may reuse the stages
                    PH(5);
                    // Diagonal block C = -acc to SMEM, then fused unblocked Cholesky + inverse.
                    if (warp < NB / 16) {
#pragma unroll
                        for (int i = 0; i < 2; ++i)
#pragma unroll
                            for (int j = 0; j < NJ; ++j)
#pragma unroll
                                for (int e = 0; e < 2; ++e) {
                                    const int rl = warp * 16 + i * 8 + g;
                                    const int nl = j * 8 + 2 * t + e;
                                    if (nl <= rl) LJ[rl * LJS + nl] = -acc[i][j][e];
                                }
                    }
                    // Blocked Cholesky of C[0:jw, 0:jw] in panels of 8 columns with the inverse
                    // built alongside (R = I - sum L Linv, rows finished panel by panel):
                    //   warp 0:   factor the panel (rsqrt pivots, register shuffles, no CTA
                    //             barrier) and finish the panel's rows of Linv;
                    //   warps 1-7, meanwhile: the previous panel's update of the far trailing
                    //             part of C and R (look-ahead);
                    //   all:      this panel's update of the next panel's columns and R rows.
                    // 16 CTA barriers per diagonal block instead of 128.
                    double *RI = LJ + NB * LJS;  // R / Linv rows, [n][q] stride LJS
                    for (int e = tid; e < NB * LJS; e += NT) RI[e] = (e / LJS == e % LJS) ? 1.0 : 0.0;
                    if (tid == 0) s_fail = 0;
                    gsync();
                    PH(12);
                    for (int p0 = 0; p0 < jw; p0 += 8) {
                        const int pw = min(8, jw - p0);
                        if (warp == 0) {
                            const int ra = p0 + lane, rb = p0 + 32 + lane;
                            double va[8], vb[8];
#pragma unroll
                            for (int c2 = 0; c2 < 8; ++c2) {
                                va[c2] = (ra < jw && c2 < pw) ? LJ[ra * LJS + p0 + c2] : 0.0;
                                vb[c2] = (NB > 32 && rb < jw && c2 < pw) ? LJ[rb * LJS + p0 + c2] : 0.0;
                            }
                            bool bad = false;
                            double rinv[8];
#pragma unroll
                            for (int c2 = 0; c2 < 8; ++c2) rinv[c2] = 0.0;
#pragma unroll
                            for (int c2 = 0; c2 < 8; ++c2) {
                                if (c2 < pw && !bad) {
                                    const double piv = __shfl_sync(0xffffffffu, va[c2], c2);
                                    // the unscaled column entries of rows p0+c3 do not depend
                                    // on the pivot: fetched while its rsqrt runs
                                    double lu[8];
#pragma unroll
                                    for (int c3 = c2 + 1; c3 < 8; ++c3) lu[c3] = __shfl_sync(0xffffffffu, va[c2], c3);
                                    if (!(piv > 0.0)) {  // not positive definite (R12); warp-uniform
                                        bad = true;
                                    } else {
                                        const double inv = rsqrt_nb(piv);
#if PGPCV_PIVOT_RCP
                                        // l / pivot from the hardware reciprocal estimate y0 and a
                                        // second-order correction folded into the multiplier:
                                        // l y0 (1 + e + e^2), e = 1 - pivot y0 -- four dependent FP64
                                        // operations from the pivot to the next one instead of
                                        // seven (rsqrt_nb, its square, the product); inv leaves
                                        // the chain (it only scales the stored column)
                                        double y0;
                                        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(piv));
                                        const double e1 = fma(-piv, y0, 1.0);
                                        const double e2 = fma(e1, e1, e1);
#pragma unroll
                                        for (int c3 = c2 + 1; c3 < 8; ++c3) {
                                            const double f0 = lu[c3] * y0;
                                            const double f = fma(e2, f0, f0);
                                            va[c3] -= va[c2] * f;
                                            vb[c3] -= vb[c2] * f;
                                        }
#else
                                        const double rp = inv * inv;  // 1 / pivot
                                        // trailing columns of the panel with the unscaled column:
                                        // (u inv)(l inv) = u l / pivot
#pragma unroll
                                        for (int c3 = c2 + 1; c3 < 8; ++c3) {
                                            const double f = lu[c3] * rp;
                                            va[c3] -= va[c2] * f;
                                            vb[c3] -= vb[c2] * f;
                                        }
#endif
                                        const double sd = piv * inv;
                                        rinv[c2] = inv;
                                        if (lane == 0) dg[p0 + c2] = sd;
                                        va[c2] = lane == c2 ? sd : (lane > c2 ? va[c2] * inv : va[c2]);
                                        vb[c2] *= inv;
                                    }
                                }
                            }
#pragma unroll
                            for (int c2 = 0; c2 < 8; ++c2) {
                                if (c2 < pw && ra < jw && lane >= c2) LJ[ra * LJS + p0 + c2] = va[c2];
                                if (NB > 32 && c2 < pw && rb < jw) LJ[rb * LJS + p0 + c2] = vb[c2];
                            }
                            if (bad && lane == 0) s_fail = 1;
                            __syncwarp();
                            // the panel's rows of Linv: Linv[r] = (R[r] - sum_{i2<i} L[r][p0+i2] Linv[p0+i2]) / L[r][r],
                            // a forward substitution in registers: lane owns columns q = lane, lane + 32
                            // of the panel's 8 rows; L[p0+i][p0+i2] comes from lane i's va[i2]
                            // (entries with q > r stay exactly 0, as Linv is lower triangular)
                            if (!bad) {
                                double w0[8], w1[8];
#pragma unroll
                                for (int i = 0; i < 8; ++i) {
                                    w0[i] = i < pw ? RI[(p0 + i) * LJS + lane] : 0.0;
                                    w1[i] = (NB > 32 && i < pw) ? RI[(p0 + i) * LJS + lane + 32] : 0.0;
                                }
#if PGPCV_PIVOT_RCP
                                // (row i pre-scaled by 1 / L_ii off the chain: one dependent
                                // operation per row instead of two)
#pragma unroll
                                for (int i = 0; i < 8; ++i) {
                                    w0[i] *= rinv[i];
                                    w1[i] *= rinv[i];
#pragma unroll
                                    for (int i2 = 0; i2 < i; ++i2) {
                                        const double l = __shfl_sync(0xffffffffu, va[i2], i) * rinv[i];
                                        w0[i] -= l * w0[i2];
                                        w1[i] -= l * w1[i2];
                                    }
                                    w0[i] = lane <= p0 + i ? w0[i] : 0.0;
                                    w1[i] = lane + 32 <= p0 + i ? w1[i] : 0.0;
                                }
#else
#pragma unroll
                                for (int i = 0; i < 8; ++i) {
#pragma unroll
                                    for (int i2 = 0; i2 < i; ++i2) {
                                        const double l = __shfl_sync(0xffffffffu, va[i2], i);
                                        w0[i] -= l * w0[i2];
                                        w1[i] -= l * w1[i2];
                                    }
                                    w0[i] = lane <= p0 + i ? w0[i] * rinv[i] : 0.0;
                                    w1[i] = lane + 32 <= p0 + i ? w1[i] * rinv[i] : 0.0;
                                }
#endif
#pragma unroll
                                for (int i = 0; i < 8; ++i) {
                                    if (i < pw && lane <= p0 + i) RI[(p0 + i) * LJS + lane] = w0[i];
                                    if (NB > 32 && i < pw && lane + 32 <= p0 + i) RI[(p0 + i) * LJS + lane + 32] = w1[i];
                                }
                            }
                        }
                        else if (p0 > 0) {
                            // Look-ahead: while warp 0 factors this panel, warps 1-7 apply the
                            // PREVIOUS panel (q0 = p0 - 8) to everything beyond this panel:
                            // C columns >= f1 and the R rows >= f1.  This panel's own columns
                            // and R rows got the previous panel in the last iteration's second
                            // phase, so the two updates touch disjoint entries.
                            // (a row per warp, columns across the lanes: no index division and
                            // no idle upper-triangle iterations)
                            const int q0 = p0 - 8, f1 = p0 + pw;
                            for (int rr = f1 + warp - 1; rr < jw; rr += NWARP - 1)
                                for (int cc = f1 + lane; cc <= rr; cc += 32) {
                                    double v = LJ[rr * LJS + cc];
#pragma unroll
                                    for (int i = 0; i < 8; ++i) v -= LJ[rr * LJS + q0 + i] * LJ[cc * LJS + q0 + i];
                                    LJ[rr * LJS + cc] = v;
                                }
                            for (int rr = f1 + warp - 1; rr < jw; rr += NWARP - 1)
                                for (int q = lane; q < p0; q += 32) {
                                    double v = RI[rr * LJS + q];
#pragma unroll
                                    for (int i = 0; i < 8; ++i) v -= LJ[rr * LJS + q0 + i] * RI[(q0 + i) * LJS + q];
                                    RI[rr * LJS + q] = v;
                                }
                        }
                        PH(13);
                        gsync();
                        if (s_fail) break;  // uniform
                        // this panel applied to the NEXT panel's columns and R rows only (all warps)
                        const int p1 = p0 + pw;
                        if (p1 < jw) {
                            const int mt = jw - p1, pn = min(8, mt);
                            // (fixed power-of-two strides instead of index divisions)
                            for (int e = tid; e < mt * 8; e += NT) {  // C[rr][cc] -= L[rr][panel] . L[cc][panel]
                                const int rr = p1 + (e >> 3), cc = p1 + (e & 7);
                                if (cc - p1 >= pn || cc > rr) continue;
                                double v = LJ[rr * LJS + cc];
                                for (int i = 0; i < pw; ++i) v -= LJ[rr * LJS + p0 + i] * LJ[cc * LJS + p0 + i];
                                LJ[rr * LJS + cc] = v;
                            }
                            for (int e = tid; e < pn * NB; e += NT) {  // R[rr][q] -= L[rr][panel] . Linv[panel][q]
                                const int rr = p1 + e / NB, q = e % NB;
                                if (q >= p1) continue;
                                double v = RI[rr * LJS + q];
                                for (int i = 0; i < pw; ++i) v -= LJ[rr * LJS + p0 + i] * RI[(p0 + i) * LJS + q];
                                RI[rr * LJS + q] = v;
                            }
                        }
                        gsync();
                        PH(14);
                    }
                    gsync();
                    if (s_fail) {
                        if (G::WS && tid == 0) add_release_u32(go, 1);  // hand-off 2 (failed: the item ends)
                        failed = true;
                        break;
                    }
                    // Linv^T for the TRSM-as-GEMM: Bt[q][n] = Linv[n][q] (zero outside the block);
                    // Linv itself is kept per block column for the back-substitution.
                    // (items that predict by bordering and do not back-substitute -- no GLS --
                    // never read the stored inverses)
                    const bool keep_linv = !(G::BORDER && nbt > 0 && np == 0);
                    for (int e = tid; e < NB * NB; e += NT) {
                        const int q = e / NB, nn = e % NB;
                        Bt[q * BS + nn] = (q <= nn && nn < jw) ? RI[nn * LJS + q] : 0.0;
                        const int rr = e / NB, cc2 = e % NB;  // Linv row-major [rr][cc2]
                        if (keep_linv)
                            linvG[(size_t)jb * NB * NB + e] = (cc2 <= rr && rr < jw) ? RI[rr * LJS + cc2] : 0.0;
                    }
                    gsync();
                    if ((a.flags & kCvNll) && warp == 0) {  // log det of this diagonal block
                        double l = 0.0;
                        for (int q = lane; q < jw; q += 32) l += log(dg[q]);
                        logdet += warp_sum(l);
                    }
                    PH(6);
                    // L_jj -> the factor (lower triangle; the diagonal from the pivots)
                    for (int rr = warp; rr < jw; rr += NWARP)  // a row per warp
                        for (int cc = lane; cc <= rr; cc += 32)
                            L[lidx(ld, j0 + rr, j0 + cc)] = rr == cc ? dg[cc] : LJ[rr * LJS + cc];
                    fence_proxy_async();  // generic LJ accesses before bulk copies refill it
                    gsync();      // LJ (stage memory) dead from here on
                    if (G::WS && tid == 0) add_release_u32(go, 1);  // hand-off 2: stages free for tile 1
                    PH(7);
                }

                // Prefetch the next row tile's first chunks (same block column: they read
                // only earlier block columns) so their latency hides behind the TRSM.
                if (!G::WS && rt + 1 < ntiles && tid == 0)
                    issued = pc + tile_prologue<G>(pc, nk, stage, full, empty, L, ld, r0 + MT, j0, (rt + 1) & 1, run_next);
                if constexpr (G::SIG) {  // the next tile's covariance entries into L2
                    if (tid == 0) {
                        if (rt + 1 < ntiles) sig_prefetch(r0 + MT, j0);
                        else if (jb + 1 < nblk) sig_prefetch(j0 + NB, j0 + NB);
                    }
                }
                __syncwarp();

                // X = C . Linv^T = -(acc . Linv^T) (triangular solve against L_jj^T as a
                // GEMM).  The A fragment for k-slice sl (columns 4sl..4sl+3) of row block i
                // is acc[g][4sl + t], held by lane 4g + 2(sl&1) + t/2 as element t&1 of
                // acc[i][sl/2].  Two passes of 32 output columns keep C (64 registers) plus
                // one half of X (32 registers) live, within the 128-register budget.
                const int rskip = rt == 0 ? j0 + jw : 0;  // first row below L_jj
                const int src_lo = (g << 2) + (t >> 1);
                const bool odd = t & 1;
#pragma unroll
                for (int h = 0; h < NB / 32; ++h) {
                    double xo[2][4][2];
#pragma unroll
                    for (int i = 0; i < 2; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) xo[i][j][0] = xo[i][j][1] = 0.0;
#pragma unroll
                    for (int sl = 0; sl < NB / 4; ++sl) {
                        const int src = src_lo + 2 * (sl & 1);
                        double af[2];
#pragma unroll
                        for (int i = 0; i < 2; ++i) {
                            const double v0 = __shfl_sync(0xffffffffu, acc[i][sl >> 1][0], src);
                            const double v1 = __shfl_sync(0xffffffffu, acc[i][sl >> 1][1], src);
                            af[i] = odd ? v1 : v0;
                        }
                        const double *bp = Bt + (sl * 4 + t) * BS + h * 32 + g;
                        double bf[4];
#pragma unroll
                        for (int j = 0; j < 4; ++j) bf[j] = bp[j * 8];
                        // Linv^T is upper triangular: B[q][n] = 0 for q > n, so k-slice
                        // sl contributes to column block jj only if 4 sl <= 8 jj + 7.
#pragma unroll
                        for (int j = 0; j < 4; ++j)
#pragma unroll
                            for (int i = 0; i < 2; ++i)
                                if (sl <= 2 * (h * 4 + j) + 1) dmma(xo[i][j], af[i], bf[j]);
                    }
                    // (columns 2t, 2t+1 of a fragment are adjacent in the swizzled layout:
                    // one 16-B store per pair)
#pragma unroll
                    for (int i = 0; i < 2; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int r = rbase + i * 8 + g;
                            const int nl = h * 32 + j * 8 + 2 * t;
                            if (r <= kb && r >= rskip && nl < jw) {
                                double *dst = L + lidx(ld, r, j0 + nl);
                                if (PGPCV_PAIR_STORE && nl + 1 < jw) {
                                    *reinterpret_cast<double2 *>(dst) = make_double2(-xo[i][j][0], -xo[i][j][1]);
                                } else {
                                    dst[0] = -xo[i][j][0];
                                    if (nl + 1 < jw) L[lidx(ld, r, j0 + nl + 1)] = -xo[i][j][1];
                                }
                            }
                        }
                }
                PH(8);
                if (rt == ntiles - 1) {
                    // The factor columns just written (generic proxy) are re-read by bulk
                    // copies (async proxy) and ld.global.cg in later block columns and the
                    // back-substitution: each writer makes its stores GPU-visible and orders
                    // them before async-proxy accesses, then the barrier.
                    __threadfence();
                    fence_proxy_async();
                    gsync();
                    if (G::WS && tid == 0) add_release_u32(go, 1);  // hand-off 3: the column is stored
                }
                PH(9);
            }
        }

        if (failed) {
            if (tid == 0) {
                const double qnan = __longlong_as_double(0x7ff8000000000000ll);
                if (a.flags & kCvPredict) a.subset_loss[oi] = qnan;
                if (a.flags & kCvNll) a.logdet[oi] = a.zz[oi] = qnan;
                a.fail[oi] = 1;
            }
            continue;
        }

        // ---------------- -2 log-likelihood (Eq.2) from the same factor ----------
        // sigma2 Sigma + tau I = sigma2 (Sigma + lambda I) = sigma2 L L^T, so
        //   log det = k log sigma2 + 2 sum log L_ii,  y^T (.)^{-1} y = ||z||^2 / sigma2,
        // with z = L^{-1} y_T the bordered row k of the factor.  The item depends on zeta
        // only through (range, lambda); the sigma2 terms are added per configuration by
        // expand_kernel, so configurations sharing (range, lambda) share this factor.
        if (a.flags & kCvNll) {
            double zz = 0.0;
            for (int cc = tid; cc < k; cc += NT) {
                const double zc = __ldcg(L + lidx(ld, k, cc));
                zz += zc * zc;
            }
            zz = warp_sum(zz);
            if (lane == 0) red[warp] = zz;
            gsync();
            if (tid == 0) {
                double q = 0.0;
                for (int w = 0; w < NWARP; ++w) q += red[w];
                a.logdet[oi] = logdet;
                a.zz[oi] = q;
            }
            gsync();
        }
        if (!(a.flags & (kCvPredict | kCvGls)) || ((a.flags & kCvPredict) && m == 0)) {
            if (tid == 0) {
                if (a.flags & kCvPredict) a.subset_loss[oi] = 0.0;  // R10: no targets
                a.fail[oi] = 0;
            }
            fence_proxy_async();
            gsync();
            continue;
        }

        // ---------------- backward substitution L^T alpha = z ----------------
        // alpha (k doubles) and the per-warp partial sums (NWARP x NB) live in the stage
        // buffers when they fit, else alpha goes to the slot's scratch after the factor.
        const bool alpha_smem = k + NWARP * NB <= STAGE_DBL;
        double *alpha = alpha_smem ? stage : L + factor_doubles(ld, (k + KC - 1) / KC);
        double *part2 = alpha_smem ? stage + STAGE_DBL - NWARP * NB : stage;
        double *tvec = cx;      // NB
        // L^T alpha = (bordered row rrow): rrow = k gives alpha = (Sigma + lambda I)^{-1} y;
        // rrow = k + 1 + q gives (Sigma + lambda I)^{-1} X[:, q] (GLS).
        auto backsub = [&](int rrow) {
        for (int jb = nblk - 1; jb >= 0; --jb) {
            const int j0 = jb * NB;
            const int jw = min(NB, k - j0);
            const int rs = j0 + jw;
            // partial t_c = sum_{r >= rs} L[r][c] alpha_r: warp w takes rows rs+w+8i, lane
            // the logical columns 2 lane, 2 lane + 1 (4 contiguous 128-B rows per warp load)
            {
                const int c0 = 2 * lane;
                const int grp = (j0 >> 4) + (c0 >> 4);
                double p0 = 0.0, p1 = 0.0;
                if (c0 < jw) {
                    for (int r = rs + warp; r < k; r += NWARP) {
                        const double ar = alpha[r];
                        const double *row = L + (size_t)(gbase(ld, grp) + r) * KC;
                        const int sw = (r & 3) << 2;
                        // columns c0, c0 + 1 are adjacent in the swizzled row: one 16-B load
                        const double2 lv = __ldcg(reinterpret_cast<const double2 *>(row + ((c0 & 15) ^ sw)));
                        p0 += lv.x * ar;
                        p1 += lv.y * ar;
                    }
                }
                if (c0 < NB) {
                    part2[warp * NB + c0] = p0;
                    part2[warp * NB + c0 + 1] = p1;
                }
            }
            gsync();
            if (tid < jw) {
                double sum = 0.0;
                for (int w = 0; w < NWARP; ++w) sum += part2[w * NB + tid];
                tvec[tid] = __ldcg(L + lidx(ld, rrow, j0 + tid)) - sum;  // z_c - L[c+1:, c] . alpha
            }
            gsync();
            // L_jj^T alpha_j = t  ->  alpha_j = Linv^T t with the block's stored inverse: a
            // parallel 64 x 64 triangular mat-vec (rows r >= c), coalesced row reads
            if (tid < jw) {
                const double *G = linvG + (size_t)jb * NB * NB + tid;
                double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
                int r = tid;
                for (; r + 3 < jw; r += 4) {
                    s0 += __ldcg(G + r * NB) * tvec[r];
                    s1 += __ldcg(G + (r + 1) * NB) * tvec[r + 1];
                    s2 += __ldcg(G + (r + 2) * NB) * tvec[r + 2];
                    s3 += __ldcg(G + (r + 3) * NB) * tvec[r + 3];
                }
                for (; r < jw; ++r) s0 += __ldcg(G + r * NB) * tvec[r];
                alpha[j0 + tid] = (s0 + s1) + (s2 + s3);
            }
            gsync();
        }
        };

        if (a.flags & kCvGls) {
            // ---------------- GLS normal-equation sums (Eq. GLS; R23) ----------
            // W_q = (Sigma + lambda I)^{-1} [y | X]_q; over the training points in the
            // subset's core: b[c] += X[i][c] W_y[i], A[c][q] += X[i][c] W_q[i].
            const double *rc = a.rects + 4 * s;
            const int W = (np + 1) * np;
            for (int q = 0; q <= np; ++q) {
                backsub(k + q);
                double accq[kMaxCovariates];
#pragma unroll
                for (int cI = 0; cI < kMaxCovariates; ++cI) accq[cI] = 0.0;
                for (int i = tid; i < k; i += NT) {
                    if (!(in_core_iv(__ldg(tx + i), rc[0], rc[1], a.xmax) &&
                          in_core_iv(__ldg(ty + i), rc[2], rc[3], a.ymax)))
                        continue;
                    const double wi = alpha[i];
#pragma unroll
                    for (int cI = 0; cI < kMaxCovariates; ++cI)
                        if (cI < np) accq[cI] += __ldg(a.tX + (toff + i) * np + cI) * wi;
                }
#pragma unroll
                for (int cI = 0; cI < kMaxCovariates; ++cI) {
                    if (cI >= np) break;  // uniform across the CTA
                    const double v = warp_sum(accq[cI]);
                    if (lane == 0) red[warp] = v;
                    gsync();
                    if (tid == 0) {
                        double t = 0.0;
                        for (int w = 0; w < NWARP; ++w) t += red[w];
                        a.gls_out[s * W + (q == 0 ? np * np + cI : cI * np + (q - 1))] = t;
                    }
                    gsync();
                }
            }
            if (tid == 0) a.fail[oi] = 0;
            fence_proxy_async();
            gsync();
            continue;
        }
        if (G::BORDER && nbt > 0) {
            // ---------------- bordered prediction (Eq.3, Eq.4): yhat_v = w_v . z ----------
            double *zs = stage;  // z = L^{-1} y_T, row k of the factor
            for (int c = tid; c < k; c += NT) zs[c] = __ldcg(L + lidx(ld, k, c));
            gsync();
            double part = 0.0;
            for (int v = warp; v < m; v += NWARP) {
                double sum = 0.0;
                for (int c = lane; c < k; c += 32) sum += __ldcg(L + lidx(ld, k + 1 + v, c)) * zs[c];
                sum = warp_sum(sum);
                if (a.yhat && lane == 0) a.yhat[voff + v] = sum;
                const double e = sum - __ldg(a.vv + voff + v);
                part += e * e;
            }
            if (lane == 0) red[warp] = part;
            fence_proxy_async();  // generic zs accesses before the next item's bulk copies
            gsync();
            if (tid == 0) {
                double l = 0.0;
                for (int w = 0; w < NWARP; ++w) l += red[w];
                a.subset_loss[oi] = l;
                a.fail[oi] = 0;
            }
            PH(11);
            continue;
        }
        backsub(k);
        PH(10);

        // ---------------- prediction and squared error (Eq.3, Eq.4) ----------------
        const double *vx = a.vx + voff, *vy = a.vy + voff, *vv = a.vv + voff;
        double part = 0.0;
        for (int v = warp; v < m; v += NWARP) {
            const double px = __ldg(vx + v), py = __ldg(vy + v);
            double sum = 0.0;
            for (int j = lane; j < k; j += 32) {
                sum += cov_exp(px - __ldg(tx + j), py - __ldg(ty + j), ninv, etab) * alpha[j];
            }
            sum = warp_sum(sum);
            if (a.yhat && lane == 0) a.yhat[voff + v] = sum;
            const double e = sum - __ldg(vv + v);
            part += e * e;
        }
        if (lane == 0) red[warp] = part;
        fence_proxy_async();  // generic alpha/part2 accesses before the next item's bulk copies
        gsync();
        if (tid == 0) {
            double l = 0.0;
            for (int w = 0; w < NWARP; ++w) l += red[w];
            a.subset_loss[oi] = l;
            a.fail[oi] = 0;
        }
        PH(11);
    }
}

// WS producer (one lane of warp 2 NWARP + g): replays its group's sequence of (item, block
// column, row tile, chunk) exactly as the consumers walk it and issues every operand chunk
// as soon as its stage is released -- no consumer warp ever waits to refill a stage (P6:
// a dedicated producer warp streams 5-6 % faster than thread 0 producing).  Hand-offs from
// the group's thread 0 (counter `go`, release/acquire): 1 an item claimed (s_item), 2 the
// diagonal block done (stage memory free again for tile 1; s_fail), 3 a block column stored
// (its factor columns are the next column's operands).  `ack` counts the items whose chunks
// were all issued; the consumers claim the next item only after it (s_item is read here).
template <class G>
__device__ void ws_producer(const CvArgs &a, double *stage, uint64_t *full, uint64_t *empty, const double *L,
                           const unsigned *go, unsigned *ack, const int *s_item, const int *s_fail) {
    constexpr int MT = G::MT, NB = G::NB;
    uint32_t pc = 0;
    unsigned seen = 0, done = 0;
    auto next = [&]() { wait_count(go, ++seen); };
    // chunks i = 0..nk-1 of row tile (r0, rev); L2 prefetch PFD chunks ahead, running on into
    // the next row tile of the block column (r0n >= 0)
    auto tile = [&](int64_t ld, int r0, int j0, int nk, bool rev, int r0n) {
        if (nk == 0) return;
        fence_proxy_async();
        for (int i = 0; i < nk; ++i) {
            issue_chunk<G>(pc + i, stage, full, empty, L, ld, r0, j0, chunk_col(i, nk, rev));
            const int ip = i + PFD;
            if (ip < nk)
                prefetch_chunk<G>(L, ld, r0, j0, chunk_col(ip, nk, rev));
            else if (r0n >= 0 && ip - nk < nk)
                prefetch_chunk<G>(L, ld, r0n, j0, chunk_col(ip - nk, nk, !rev));
        }
        pc += nk;
    };
    for (;;) {
        next();  // 1
        const int item = *(volatile const int *)s_item;
        if (item >= a.n_items) return;
        const int s = a.items[item].x;
        const int k = (int)(a.train_off[s + 1] - a.train_off[s]);
        const int m = (int)(a.val_off[s + 1] - a.val_off[s]);
        const int np = (a.flags & kCvGls) ? a.p : 0;
        const int nbt = G::BORDER ? (int)border_rows(a.flags, a.border_pred, k, m) : 0;
        const int kb = k + np + nbt;
        const int64_t ld = factor_ld(kb);
        const int nblk = (k + NB - 1) / NB;
        bool failed = false;
        for (int jb = 0; jb < nblk; ++jb) {
            const int j0 = jb * NB;
            const int ntiles = (kb + 1 - j0 + MT - 1) / MT;
            const int nk = j0 / KC;
            if (jb > 0) next();  // 3 (previous column)
            for (int i = 0; i < min(PFD, nk); ++i) prefetch_chunk<G>(L, ld, j0, j0, chunk_col(i, nk, false));
            tile(ld, j0, j0, nk, false, ntiles > 1 ? j0 + MT : -1);
            next();  // 2
            if (*(volatile const int *)s_fail) {
                failed = true;
                break;
            }
            for (int rt = 1; rt < ntiles; ++rt)
                tile(ld, j0 + rt * MT, j0, nk, rt & 1, rt + 1 < ntiles ? j0 + (rt + 1) * MT : -1);
        }
        if (!failed && nblk > 0) next();  // 3 (last column; k = 0 has none)
        add_release_u32(ack, 1);
        ++done;
    }
}

// K4s sigma_kernel: Sigma_theta(s) = exp(-D_s / theta) for every small subset s of the call
// and every distinct range theta of its configurations (Eq.3).  The covariance
// depends on a configuration only through the range; lambda = nugget / sigma2 moves only the
// diagonal, so the (range, lambda) items of one subset read these entries instead of
// each regenerating the k^2/2 distances and exponentials (BASELINE north_star: distances
// reused across parameter configurations).  kSigmaSplit CTAs per (subset, range), CTA p taking
// column groups p, p + kSigmaSplit, ... (the call's subsets fill the GPU even at c2's 100), writing the block
// in the factor's packed, swizzled column-group layout with ld = sigma_ld(k, nbt): rows
// 0..k-1 the training points, rows k+1..k+nbt the bordered targets' cross-covariance, row k
// (y) and entries above the diagonal or past column k zero.  Writes are fully coalesced
// (consecutive threads, consecutive doubles); HBM-write-bound at 8 B per entry.
constexpr int kSigmaSplit = 8;
__global__ void __launch_bounds__(256) sigma_kernel(const int32_t *subs, int32_t n_subs, const double *ranges,
                                                    const int64_t *train_off, const int64_t *val_off,
                                                    const double *tx, const double *ty, const double *vx,
                                                    const double *vy, int32_t flags, int32_t border_pred,
                                                    double *sig, const int64_t *sig_off, size_t sig_stride) {
    __shared__ double etab[EXP_TAB];
    if (threadIdx.x < EXP_TAB) etab[threadIdx.x] = kExp2Tab[threadIdx.x];
    __syncthreads();
    const int part = blockIdx.x % kSigmaSplit;
    const int s = subs[(blockIdx.x / kSigmaSplit) % n_subs];
    const int ri = blockIdx.x / kSigmaSplit / n_subs;
    const int64_t toff = train_off[s], voff = val_off[s];
    const int k = (int)(train_off[s + 1] - toff);
    const int m = (int)(val_off[s + 1] - voff);
    const int nbt = (int)border_rows(flags, border_pred, k, m);
    const int64_t ld = sigma_ld(k, nbt);
    const double ninv = -1.0 / ranges[ri];  // the kernel's own division (bit-identical)
    double *out = sig + (size_t)ri * sig_stride + sig_off[s];
    const double *px = tx + toff, *py = ty + toff, *qx = vx + voff, *qy = vy + voff;
    const int groups = (k + KC - 1) / KC;
    for (int q = part; q < groups; q += kSigmaSplit) {
        const int64_t n = (ld - 16 * q) * KC;
        double *blk = out + (size_t)(gbase(ld, q) + 16 * q) * KC;
        for (int64_t idx = threadIdx.x; idx < n; idx += blockDim.x) {
            const int r = 16 * q + (int)(idx >> 4);
            const int c = 16 * q + ((int)(idx & 15) ^ ((r & 3) << 2));
            double v = 0.0;
            if (c < k) {
                if (r < k && r >= c)
                    v = cov_exp(__ldg(px + r) - __ldg(px + c), __ldg(py + r) - __ldg(py + c), ninv, etab);
                else if (r > k && r <= k + nbt)
                    v = cov_exp(__ldg(qx + (r - k - 1)) - __ldg(px + c), __ldg(qy + (r - k - 1)) - __ldg(py + c),
                                ninv, etab);
            }
            blk[idx] = v;
        }
    }
}

// out[c] = sum_s vals[s, c] in ascending s (Alg.1 line 9) over the subsets the
// mask admits (mask_off[s+1] > mask_off[s], i.e. subsets with targets; all when null);
// status[c] = the smallest failing admitted subset or -1.  One CTA per config: the threads
// stage a chunk of the strided column vals[:, c] in SMEM (independent loads in flight
// together; a single thread walking the column paid one L2 round trip per subset, ~0.9 ms at
// c5's 2,500 subsets), then thread 0 adds the chunk in ascending s -- the same fixed,
// deterministic order as before, bit for bit.  Entries that are not admitted or failed are
// staged as +0.0, which leaves the running sum unchanged (it starts at +0.0, so it is never
// -0.0); a failed admitted entry makes the result NaN anyway.
constexpr int kReduceChunk = 2048;
__global__ void __launch_bounds__(256) reduce_kernel(const double *vals, const uint8_t *fail, const int64_t *mask_off,
                                                     int64_t N, int32_t C, double *out, int32_t *status) {
    __shared__ double sv[kReduceChunk];
    __shared__ int s_first;
    const int c = blockIdx.x;
    if (threadIdx.x == 0) s_first = INT_MAX;
    double acc = 0.0;
    for (int64_t base = 0; base < N; base += kReduceChunk) {
        const int n = (int)(N - base < kReduceChunk ? N - base : kReduceChunk);
        __syncthreads();  // s_first initialised / the previous chunk summed
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const int64_t s = base + i;
            const bool admitted = !mask_off || mask_off[s + 1] != mask_off[s];
            const bool f = admitted && fail[s * C + c];
            if (f) atomicMin(&s_first, (int)s);
            sv[i] = admitted && !f ? vals[s * C + c] : 0.0;
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int i = 0; i < n; ++i) acc += sv[i];
    }
    if (threadIdx.x == 0) {
        const int64_t st = s_first == INT_MAX ? -1 : s_first;
        out[c] = st >= 0 ? __longlong_as_double(0x7ff8000000000000ll) : acc;
        if (status) status[c] = (int32_t)st;
    }
}

// zeta dedup (pgpcv_evaluate): every configuration c takes the results of its unique
// (range, lambda) u = umap[c]; the likelihood adds the sigma2 terms of Eq.2,
//   -2 log L = k log 2pi + k log sigma2 + 2 sum log L_ii + ||z||^2 / sigma2.
// Subsets this rank did not evaluate hold exact zeros (a sum over ranks is then exact).
__global__ void expand_kernel(int64_t N, int32_t C, int32_t U, const int32_t *umap, const uint8_t *own,
                              const int64_t *train_off, const double *sigma2, const double *u_loss,
                              const uint8_t *u_fail, const double *u_logdet, const double *u_zz, double *loss,
                              uint8_t *fail, double *nll) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N * C; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = e / C;
        const int c = (int)(e - s * C);
        const int64_t ue = s * U + umap[c];
        if (!own[s]) {
            loss[e] = 0.0;
            fail[e] = 0;
            if (nll) nll[e] = 0.0;
            continue;
        }
        loss[e] = u_loss[ue];
        fail[e] = u_fail[ue];
        if (nll) {
            const double kd = (double)(train_off[s + 1] - train_off[s]);
            const double s2 = sigma2[c];
            nll[e] = u_fail[ue] ? __longlong_as_double(0x7ff8000000000000ll)
                                : kd * log(2.0 * 3.14159265358979323846) + kd * log(s2) + 2.0 * u_logdet[ue] +
                                      u_zz[ue] / s2;
        }
    }
}

// Diagnostic: the elementary functions exactly as cv_kernel inlines them.
__global__ void device_math_kernel(int32_t fn, int64_t n, const double *x, double *y) {
    __shared__ double etab[EXP_TAB];
    if (threadIdx.x < EXP_TAB) etab[threadIdx.x] = kExp2Tab[threadIdx.x];
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = x[i];
        y[i] = fn == 0 ? exp_neg(v, etab) : (fn == 1 ? sqrt_nb(v) : rsqrt_nb(v));
    }
}

// GLS: W = (p+1) p entries per subset; thread w sums entry w over subsets in ascending s
// (failed subsets poison the sums), then thread 0 solves A beta = b by Gaussian elimination
// with partial pivoting (largest |pivot|, first on ties).
__global__ void gls_solve_kernel(const double *part, const uint8_t *fail, int64_t N, int32_t p, double *sums,
                                 double *beta, int32_t *status) {
    const int W = (p + 1) * p;
    for (int w = threadIdx.x; w < W; w += blockDim.x) {
        double acc = 0.0;
        for (int64_t s = 0; s < N; ++s) acc += fail[s] ? __longlong_as_double(0x7ff8000000000000ll) : part[s * W + w];
        sums[w] = acc;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    double A[kMaxCovariates * kMaxCovariates], b[kMaxCovariates];
    for (int i = 0; i < p * p; ++i) A[i] = sums[i];
    for (int i = 0; i < p; ++i) b[i] = sums[p * p + i];
    int32_t st = 0;
    for (int c = 0; c < p && !st; ++c) {
        int piv = c;
        for (int r = c + 1; r < p; ++r)
            if (fabs(A[r * p + c]) > fabs(A[piv * p + c])) piv = r;
        if (!(A[piv * p + c] != 0.0)) {
            st = 1;
            break;
        }
        if (piv != c) {
            for (int j = 0; j < p; ++j) {
                const double t = A[c * p + j];
                A[c * p + j] = A[piv * p + j];
                A[piv * p + j] = t;
            }
            const double t = b[c];
            b[c] = b[piv];
            b[piv] = t;
        }
        for (int r = c + 1; r < p; ++r) {
            const double f = A[r * p + c] / A[c * p + c];
            for (int j = c; j < p; ++j) A[r * p + j] -= f * A[c * p + j];
            b[r] -= f * b[c];
        }
    }
    for (int r = p - 1; r >= 0; --r) {
        double sum = b[r];
        for (int j = r + 1; j < p; ++j) sum -= A[r * p + j] * beta[j];
        beta[r] = st ? __longlong_as_double(0x7ff8000000000000ll) : sum / A[r * p + r];
    }
    *status = st;
}

__global__ void gather_rows_kernel(int64_t cnt, const int32_t *idx, const double *X, int32_t p, double *out) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < cnt * p;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / p;
        out[e] = X[(int64_t)idx[i] * p + (e - i * p)];
    }
}

}  // namespace

cudaError_t launch_gls_solve(const double *part, const uint8_t *fail, int64_t N, int32_t p, double *sums,
                             double *beta, int32_t *status, cudaStream_t st) {
    gls_solve_kernel<<<1, 128, 0, st>>>(part, fail, N, p, sums, beta, status);
    return cudaGetLastError();
}

cudaError_t launch_gather_rows(int64_t cnt, const int32_t *idx, const double *X, int32_t p, double *out,
                               cudaStream_t st) {
    if (cnt == 0) return cudaSuccess;
    const int64_t total = cnt * p;
    const int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 32);
    gather_rows_kernel<<<grid, 256, 0, st>>>(cnt, idx, X, p, out);
    return cudaGetLastError();
}

template <class G>
size_t slot_doubles(int64_t kmax, int extra_rows) {
    // the packed factor + alpha when it does not fit in SMEM + the inverse of every diagonal
    // block + MT x 16: a bulk copy of the last group's row tile may read past the factor's
    // end.  Rounded to 256 B so every slot base keeps the alignment bulk copies need.
    const int64_t groups = (kmax + KC - 1) / KC;
    const size_t d = (size_t)factor_doubles(factor_ld(kmax + extra_rows), groups > 0 ? groups : 1) +
                     (size_t)((kmax + 31) / 32) * 32 + (size_t)((kmax + G::NB - 1) / G::NB) * G::NB * G::NB +
                     (size_t)G::MT * KC;
    return (d + 31) / 32 * 32;
}

template <class G>
cudaError_t occupancy(int *blocks_per_sm) {
    cudaError_t e = cudaFuncSetAttribute(cv_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)G::CTA_SMEM);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, cv_kernel<G>, G::THREADS, G::CTA_SMEM);
    *blocks_per_sm *= G::GROUPS;  // factor slots (item streams) per SM
    return e;
}

template <class G>
cudaError_t launch(const CvArgs &a, int grid, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(cv_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)G::CTA_SMEM);
    if (e != cudaSuccess) return e;
    // `grid` counts factor slots; a WS CTA serves GROUPS of them (the host rounds up)
    cv_kernel<G><<<(grid + G::GROUPS - 1) / G::GROUPS, G::THREADS, G::CTA_SMEM, st>>>(a);
    return cudaGetLastError();
}

// dispatch on the kernel variant (kCv*)
template <class F>
auto with_geo(int variant, F f) {
    switch (variant) {
        case kCvSmall: return f(GeoSmall{});
        case kCvSmallSig: return f(GeoSmallSig{});
        case kCvLargeWS: return f(GeoLargeWS{});
        default: return f(GeoLarge{});
    }
}
size_t cv_kernel_smem_bytes(int variant) {
    return with_geo(variant, [](auto g) { return decltype(g)::CTA_SMEM; });
}
int cv_kernel_slots_per_cta(int variant) {
    return with_geo(variant, [](auto g) { return decltype(g)::GROUPS; });
}
int cv_kernel_max_k() { return PGPCV_MAX_K_INTERNAL; }  // = PGPCV_MAX_K (include/pgpcv.h)
size_t cv_kernel_slot_doubles(int variant, int64_t kmax, int extra_rows) {
    return with_geo(variant, [&](auto g) { return slot_doubles<decltype(g)>(kmax, extra_rows); });
}
cudaError_t cv_kernel_occupancy(int variant, int *blocks_per_sm) {
    return with_geo(variant, [&](auto g) { return occupancy<decltype(g)>(blocks_per_sm); });
}
cudaError_t launch_cv_kernel(int variant, const CvArgs &a, int grid, cudaStream_t st) {
    return with_geo(variant, [&](auto g) { return launch<decltype(g)>(a, grid, st); });
}

cudaError_t launch_expand(int64_t N, int32_t C, int32_t U, const int32_t *umap, const uint8_t *own,
                          const int64_t *train_off, const double *sigma2, const double *u_loss,
                          const uint8_t *u_fail, const double *u_logdet, const double *u_zz, double *loss,
                          uint8_t *fail, double *nll, cudaStream_t st) {
    if (N * C == 0) return cudaSuccess;
    const int grid = (int)std::min<int64_t>((N * C + 255) / 256, 148 * 8);
    expand_kernel<<<grid, 256, 0, st>>>(N, C, U, umap, own, train_off, sigma2, u_loss, u_fail, u_logdet, u_zz, loss,
                                        fail, nll);
    return cudaGetLastError();
}

int64_t sigma_doubles(int64_t k, int64_t nbt) {
    const int64_t groups = (k + KC - 1) / KC;
    return groups > 0 ? factor_doubles(sigma_ld(k, nbt), groups) : 0;
}

cudaError_t launch_sigma(const int32_t *subs, int32_t n_subs, const double *ranges, int32_t n_ranges,
                         const int64_t *train_off, const int64_t *val_off, const double *tx, const double *ty,
                         const double *vx, const double *vy, int32_t flags, int32_t border_pred, double *sig,
                         const int64_t *sig_off, size_t sig_stride, cudaStream_t st) {
    if ((int64_t)n_subs * n_ranges == 0) return cudaSuccess;
    sigma_kernel<<<(unsigned)((int64_t)n_subs * n_ranges * kSigmaSplit), 256, 0, st>>>(subs, n_subs, ranges, train_off, val_off, tx,
                                                                         ty, vx, vy, flags, border_pred, sig, sig_off,
                                                                         sig_stride);
    return cudaGetLastError();
}

cudaError_t launch_device_math(int32_t fn, int64_t n, const double *x, double *y, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    device_math_kernel<<<grid, 256, 0, st>>>(fn, n, x, y);
    return cudaGetLastError();
}

cudaError_t launch_reduce(const double *vals, const uint8_t *fail, const int64_t *mask_off, int64_t N,
                          int32_t C, double *out, int32_t *status, cudaStream_t st) {
    if (C <= 0) return cudaSuccess;
    reduce_kernel<<<C, 256, 0, st>>>(vals, fail, mask_off, N, C, out, status);
    return cudaGetLastError();
}

}  // namespace pgpcv
