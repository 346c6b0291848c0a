/*
 * pgpcv.h -- C ABI of libpgpcv: the data-parallel hot path of parallel cross-validation
 * for Gaussian-process models (Gerber & Nychka, "Parallel cross-validation: a scalable
 * fitting method for Gaussian process models", arXiv 1912.13132) on NVIDIA B200 (sm_100a).
 *
 * Citations: P:n = PAPER.md line n (LaTeX source of the paper); R# = reading number in
 * DESIGN.md (where the paper is silent, the reading taken).
 *
 * The library evaluates, for every parameter configuration zeta = (range, sigma2, nugget),
 *
 *     C~V(y_T, y_V, zeta) = sum_{i=1..N} CV(y~^i_T, y^i_V, zeta)                 Eq.7
 *     CV(y_T, y_V, zeta)  = sum_v (yhat_v - y_v)^2                                Eq.4
 *     yhat_p = Sigma_p^T (Sigma + lambda I)^{-1} y,  lambda = nugget / sigma2    Eq.3
 *     Sigma_ij = exp(-||s_i - s_j|| / range)                                      Sec.3
 *
 * as Algorithm 1 does: the data are divided into subsets once
 * (pgpcv_partition, Alg.1 lines 2-3), each subset's local SSPE z_i is computed
 * (pgpcv_cv_loss, lines 4-8) and the z_i are combined (line 9; across GPUs by one NCCL
 * all-reduce after pgpcv_shard).
 *
 * Conventions for every entry point:
 *   - Return value: PGPCV_OK (0) or a negative PGPCV_E* code; no exception or abort
 *     crosses the ABI.  pgpcv_last_error(ctx) returns a message for the last failure.
 *   - Host pointers are caller-owned and only read/written for the duration of the call
 *     (the library copies in/out).  Device pointers (the *_device variants) must be
 *     memory of the ctx's CUDA device and stay valid for the duration of the call.
 *   - A ctx owns all of its device memory, its CUDA stream and its NCCL communicator.
 *     One ctx per process per GPU; a ctx is not thread-safe.
 *   - Floating point is IEEE binary64 throughout (the paper's R arithmetic).
 */
#ifndef PGPCV_H
#define PGPCV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PGPCV_VERSION 5

/* Error codes. */
#define PGPCV_OK 0
#define PGPCV_EINVAL (-2)   /* NaN/Inf input, point outside domain, range<=0, sigma2<=0,
                               nugget<0, delta<0, kx or ky < 1, n >= 2^31, bad role byte,
                               a subset larger than PGPCV_MAX_K, NULL where required */
#define PGPCV_ENUMERIC (-3) /* some (subset, config) was not positive definite (a pivot <= 0
                               or NaN in the Cholesky, R12): loss[c] = NaN and status[c] = the
                               first such subset; all other configs are valid */
#define PGPCV_EEMPTY (-4)   /* every subset lacks validation data: the loss is undefined */
#define PGPCV_ECUDA (-5)    /* CUDA runtime or launch failure */
#define PGPCV_ENOMEM (-6)   /* device or host allocation failed */
#define PGPCV_ENCCL (-7)    /* NCCL unavailable or a collective failed */
#define PGPCV_ESTATE (-8)   /* cv_loss before partition, or shard after cv_loss */

/* Largest training subset pgpcv_cv_loss accepts: one resident factorization of k points
 * holds the packed lower triangle, ~4 k^2 bytes (k = 65,536: 17 GB), and the library
 * lowers the number of resident factorizations until they fit in device memory
 * (ENOMEM when even one does not). */
#define PGPCV_MAX_K 65536

/* Point roles (R7): 0 = training (y_T), 1 = validation (y_V), 2 = test (ignored). */
#define PGPCV_ROLE_TRAIN 0
#define PGPCV_ROLE_VALIDATION 1
#define PGPCV_ROLE_TEST 2

typedef struct pgpcv_ctx pgpcv_ctx; /* opaque */

/* Rectangular domain D: [xmin, xmax] x [ymin, ymax]; tiles are half-open
 * with the domain's top edges closed (R3). */
typedef struct {
    double xmin, xmax, ymin, ymax;
} pgpcv_rect;

/* One covariance configuration in BASELINE order; only lambda = nugget / sigma2 and
 * range enter the prediction (R8). range > 0, sigma2 > 0, nugget >= 0. */
typedef struct {
    double range, sigma2, nugget;
} pgpcv_param;

/* Summary of a partition (sizes of Alg.1's y~^i_T and y^i_V). */
typedef struct {
    int64_t n_subsets;   /* N = kx * ky */
    int64_t sum_k;       /* total training memberships, sum_i |y~^i_T| */
    int64_t sum_m;       /* total validation memberships, sum_i |y^i_V| (= n_V) */
    int64_t max_k;       /* largest training subset (the paper's k) */
    int64_t max_m;       /* largest validation subset */
    int64_t n_empty_val; /* subsets with no validation data (loss 0, "ignored") */
    int64_t n_train;     /* points with role 0 */
    int64_t n_val;       /* points with role 1 */
    int64_t n_test;      /* points with role 2 (each in exactly one core tile) */
    int64_t max_test;    /* largest test subset */
} pgpcv_partition_info;

/* Outputs of pgpcv_evaluate: caller-owned host arrays, each NULL to skip it.  C = n_params,
 * N = number of subsets.  Requesting loss or subset_loss runs the CV prediction (Eq.3-4);
 * requesting nll or subset_nll adds the -2 log-likelihood (Eq.2) of every subset's
 * training data from the same factorization (no second factorization). */
typedef struct {
    double *loss;        /* [C] C~V per config (Eq.7), summed over subsets in ascending s */
    double *subset_loss; /* [N*C] subset-major SSPE z_{s,c}; exactly 0 when m_s = 0 (R10) */
    int32_t *status;     /* [C] -1 ok, else the smallest subset whose factorization failed */
    double *nll;         /* [C] sum over subsets of -2 log L_s (a composite likelihood) */
    double *subset_nll;  /* [N*C] -2 log L_s = k log(2 pi) + log det(s2 Sigma + tau I)
                            + y^T (s2 Sigma + tau I)^{-1} y over subset s's training data
                            (Eq.2); 0 when k_s = 0 */
} pgpcv_outputs;

/* Device-side timing of the last pgpcv_cv_loss call (CUDA events on the ctx stream). */
typedef struct {
    double kernel_ms;     /* the dominant kernel (batched Cholesky/solve/predict) */
    double total_ms;      /* whole call: kernels + reduction + collective + result copy */
    double flops;         /* algorithmic FP64 flops this rank executed */
    int64_t n_evals;      /* (subset, config) evaluations this rank executed (m > 0 only) */
    int32_t launches;     /* number of libpgpcv kernel launches in the call */
    int32_t n_slots;      /* resident CTAs (factorization slots) of the dominant kernel */
    int32_t n_configs_executed; /* configurations factored: pgpcv_evaluate factors each
                                   bit-identical (range, lambda) pair once */
    int32_t reserved;
} pgpcv_timing;

/* Library version (PGPCV_VERSION).  Never fails; needs no GPU. */
int pgpcv_version(void);

/* Create a context on CUDA device `cuda_device` (>= 0).  Creates a non-blocking stream.
 * *out receives the handle (NULL on failure).  Errors: EINVAL (bad device / NULL out),
 * ECUDA (no device or no sm_100 device), ENOMEM. */
int pgpcv_create(int cuda_device, pgpcv_ctx **out);

/* Release every device buffer, the stream (if owned) and the NCCL communicator.  NULL is
 * a no-op. */
void pgpcv_destroy(pgpcv_ctx *ctx);

/* Message for the last non-zero return on ctx ("" if none).  Owned by ctx; valid until
 * the next call on ctx.  ctx == NULL returns the message of the last failed
 * pgpcv_create. */
const char *pgpcv_last_error(const pgpcv_ctx *ctx);

/* Use `stream` (a cudaStream_t of the ctx device, e.g. torch's current stream) for all
 * later work; NULL restores the ctx's own stream.  The caller keeps ownership. */
int pgpcv_set_stream(pgpcv_ctx *ctx, void *stream);

/* Alg.1 lines 2-3, once per dataset: divide the n points into N = kx*ky
 * subsets (R1: equal tiles).  Subset s = iy*kx + ix (R5).
 *   training list  y~^s_T = {p : role[p] = 0 and p in the tile's L-inf dilation by
 *                            delta, clipped to D}          (shell; R2, R3, R4)
 *   validation list y^s_V = {p : role[p] = 1 and p in the core tile}    (Eq.7; R6)
 * Both lists are in ascending point index.  Membership is decided by exact FP64
 * comparisons against tile edges e_i = xmin + i*w (w = (xmax-xmin)/kx, no FMA, e_kx =
 * xmax) and dilated bounds e_i - delta, e_{i+1} + delta; it is bit-exact and identical on
 * every rank.  The member coordinates/values are then staged subset-contiguously in HBM,
 * where they stay for every later pgpcv_cv_loss call.
 *   x, y, value: float64[n] host arrays (SoA); role: uint8[n] host array.
 *   info_out: may be NULL.
 * Replaces any previous partition.  Errors: EINVAL, ECUDA, ENOMEM. */
int pgpcv_partition(pgpcv_ctx *ctx, int64_t n, const double *x, const double *y,
                    const double *value, const uint8_t *role, pgpcv_rect domain, int32_t kx,
                    int32_t ky, double delta, pgpcv_partition_info *info_out);

/* Same as pgpcv_partition with x, y, value, role already in device memory of the ctx
 * device (no host-to-device copy of the points). */
int pgpcv_partition_device(pgpcv_ctx *ctx, int64_t n, const double *d_x, const double *d_y,
                           const double *d_value, const uint8_t *d_role, pgpcv_rect domain,
                           int32_t kx, int32_t ky, double delta,
                           pgpcv_partition_info *info_out);

/* Row f2: the paper's own division -- recursive shell-balanced bisection of D
 * into N = 2^depth rectangles, then the same membership rules as pgpcv_partition (training
 * = role 0 in the rectangle's L-inf dilation by delta, validation/test = role 1/2 in the
 * rectangle).  Node 1 is D; a node at depth d is split along x (d even) or y (d odd) by the
 * line c minimising |count_left - count_right|, a child's count being the number of role 0
 * and role 1 points in its dilation by delta ("both rectangles together with their shells
 * contain a similar amount of data"); candidates are c = 0.5 (u_j + u_{j+1}) over
 * consecutive distinct split coordinates of counted points in the node, ties to the
 * smallest c, no candidate -> the node's midpoint (R19-R21).  Subset s is leaf
 * 2^depth + s of the heap-numbered tree (left = lower coordinates).
 *   depth: 0..20.
 *   shell_cap: < 0 for none; else, in every subset whose shell (training points outside
 *     its rectangle) exceeds shell_cap, keep the shell_cap shell points with the smallest
 *     keys splitmix64(seed, s * 2^32 + p + 1) (ties: smaller p), as the paper's 5M-point
 *     fit reduces shells to 2,000 "by random sampling" (R22).
 * Bit-exact and deterministic (exact FP64 comparisons, single correctly rounded ops).
 * Errors: EINVAL, ECUDA, ENOMEM. */
int pgpcv_partition_bisect(pgpcv_ctx *ctx, int64_t n, const double *x, const double *y,
                           const double *value, const uint8_t *role, pgpcv_rect domain,
                           int32_t depth, double delta, int64_t shell_cap, uint64_t seed,
                           pgpcv_partition_info *info_out);

/* Same with x, y, value, role in device memory of the ctx device. */
int pgpcv_partition_bisect_device(pgpcv_ctx *ctx, int64_t n, const double *d_x,
                                  const double *d_y, const double *d_value,
                                  const uint8_t *d_role, pgpcv_rect domain, int32_t depth,
                                  double delta, int64_t shell_cap, uint64_t seed,
                                  pgpcv_partition_info *info_out);

/* The N subset rectangles of the current partition, (x0, x1, y0, y1) per subset into the
 * caller's double[4*N] (tiles for pgpcv_partition, leaves for the bisection).
 * Errors: EINVAL (NULL), ESTATE (no partition). */
int pgpcv_partition_rects(pgpcv_ctx *ctx, double *rects);

/* Copy the CSR membership of the current partition to caller-allocated host arrays:
 * train_off int64[N+1], train_idx int32[sum_k], val_off int64[N+1], val_idx int32[sum_m]
 * (sizes from pgpcv_partition_info).  Any pointer may be NULL to skip it.
 * Errors: ESTATE (no partition), ECUDA. */
int pgpcv_partition_export(pgpcv_ctx *ctx, int64_t *train_off, int32_t *train_idx,
                           int64_t *val_off, int32_t *val_idx);

/* Multi-GPU (Alg.1's parfor over subsets, across the GPUs of one box).
 * rank in [0, world); world >= 1.  nccl_unique_id: NCCL_UNIQUE_ID_BYTES (128) bytes from
 * pgpcv_nccl_get_unique_id on rank 0, broadcast by the caller; ignored (may be NULL) when
 * world == 1.  Creates the NCCL communicator (collective over the `world` ranks).  Every
 * later evaluation assigns the whole subsets it factors to ranks by LPT on the cost k_s^3
 * (pgpcv_lpt_assign; ties by subset id), identically on every rank, and combines the
 * results with NCCL all-reduces.  Must be called after pgpcv_partition and before the
 * first evaluation of that partition (else ESTATE), or again after a collective failed.
 * Without it a ctx owns every subset.  The sharding stays in effect for later partitions of
 * the same ctx (each rank must then partition the same data).  On any error the ctx is
 * left at rank 0 of world 1
 * (no communicator).  Errors: EINVAL (bad rank/world, world > 1 without an id), ESTATE,
 * ENCCL (libnccl not loadable, ncclCommInitRank failed).
 *
 * Failure behaviour at world > 1: every rank-local failure (allocation, launch) is agreed
 * on by all ranks (one MAX all-reduce of an error flag) before any data collective, so
 * peers return ENCCL instead of blocking.  While waiting on a collective the library polls
 * ncclCommGetAsyncError; an NCCL error, or no completion within PGPCV_NCCL_TIMEOUT_S
 * seconds (environment, default 1800: a hung or dead peer), aborts the communicator
 * (ncclCommAbort) and returns ENCCL; the ctx then needs pgpcv_shard again. */
int pgpcv_shard(pgpcv_ctx *ctx, int rank, int world, const void *nccl_unique_id);

/* Which libnccl the library bound: the file named by the environment variable
 * PGPCV_NCCL_LIB when set (bound first and privately, RTLD_LOCAL -- an explicit choice,
 * e.g. the tests' host-memory stand-in), else an NCCL already loaded in the process (e.g.
 * torch's, so one process never holds two), else libnccl.so.2.  Writes "path (NCCL x.y.z)"
 * into buf[len], or the reason none could be loaded.  Needs no ctx.  Errors: EINVAL (NULL /
 * len < 1), ENCCL (no usable libnccl; buf holds the reason). */
int pgpcv_nccl_library(char *buf, int64_t len);

/* Fill `out` (NCCL_UNIQUE_ID_BYTES bytes) with a fresh ncclUniqueId.  Needs no ctx.
 * Errors: ENCCL (libnccl.so.2 not loadable), EINVAL (NULL). */
int pgpcv_nccl_get_unique_id(void *out);

/* Alg.1 lines 4-9 for n_params configurations (data resident, parameters streamed;
 * P:200): for every owned subset with validation data and every config, assemble
 * Sigma + lambda I from pairwise distances, factor it (FP64 Cholesky), solve, predict the
 * subset's validation points and sum squared errors; then combine.
 *   params: host array [n_params].
 *   loss:   host double[n_params] (required): global C~V per config (SSPE, not RMSPE),
 *           summed over all subsets (across ranks when world > 1).
 *   subset_loss: host double[N * n_params] subset-major (entry s*n_params + c), or NULL.
 *           Subsets without validation data hold exactly 0 (R10).  When world > 1 the
 *           per-subset array is all-reduced (each entry has one owner), which also makes
 *           loss[] bit-identical for every world size.
 *   status: host int32[n_params] or NULL: -1 if config c succeeded, else the smallest
 *           subset id whose factorization failed (loss[c] = NaN then).
 * Errors: EINVAL (bad params), ESTATE (no partition), EEMPTY (no validation data at all),
 * ENUMERIC (some config failed; others valid), ECUDA, ENOMEM, ENCCL. */
int pgpcv_cv_loss(pgpcv_ctx *ctx, const pgpcv_param *params, int32_t n_params, double *loss,
                  double *subset_loss, int32_t *status);

/* The general form of pgpcv_cv_loss (Alg.1 lines 4-9 plus row f3 of the scope table):
 * one batched factorization per (owned subset, config) serves every requested output.
 * Subsets enter the CV outputs when they have validation data; with nll/subset_nll
 * requested every owned subset is factored (the likelihood needs no targets).  Across
 * GPUs the [loss | nll] vector is all-reduced once (per-subset arrays, when requested,
 * are all-reduced instead; each entry has one owner so the sums are exact).
 * Errors: EINVAL (no output requested, bad params), ESTATE, EEMPTY (CV output requested
 * but no validation data), ENUMERIC (loss/nll[c] = NaN and status[c] >= 0 for a non-PD
 * config; others valid), ECUDA, ENOMEM, ENCCL. */
int pgpcv_evaluate(pgpcv_ctx *ctx, const pgpcv_param *params, int32_t n_params,
                   const pgpcv_outputs *out);

/* Grid-search consumer of the last CV evaluation (scope row f1).  Reads
 * the per-subset losses left on the device by the last pgpcv_evaluate/pgpcv_cv_loss (which
 * must have computed every subset: world 1, or subset_loss requested; else ESTATE).
 * Outputs (host, caller-owned, each NULL to skip):
 *   best:        int32[1] argmin_c loss[c] (zeta_hat_CV; ties -> lowest c; NaN
 *                configs never win; -1 if every config failed)
 *   rmspe:       double[C] global RMSPE sqrt(loss[c] / n_V)
 *   local_best:  int32[N] argmin_c subset_loss[s, c] (ties -> lowest c; -1 when m_s = 0)
 *   local_rmspe: double[N*C] sqrt(subset_loss[s, c] / m_s) (NaN when m_s = 0 or failed)
 *   wins:        int32[C] number of subsets whose local best is c
 * Errors: ESTATE, ECUDA. */
int pgpcv_select(pgpcv_ctx *ctx, int32_t *best, double *rmspe, int32_t *local_best,
                 double *local_rmspe, int32_t *wins);

/* Kriging prediction of held-out points with a chosen configuration per subset (P:466-468:
 * "the hold-out test data are predicted using the global zeta_hat_CV and using the best
 * local parameter configuration for each subset").  For every owned subset s with targets,
 * factor Sigma + lambda I of its training data y~^s_T under params[subset_config[s]]
 * (params[0] for every subset when subset_config is NULL) and predict its core-tile points
 * of role `target_role` (PGPCV_ROLE_TEST or PGPCV_ROLE_VALIDATION; with VALIDATION and one
 * config this reproduces pgpcv_cv_loss).
 *   yhat:        double[n_targets] or NULL: predictions in the target CSR order (subset-
 *                major, ascending point index; see pgpcv_partition_export_test / _export)
 *   subset_sspe: double[N] or NULL: sum of squared prediction errors per subset
 *   sspe:        double[1] or NULL: their sum in ascending s (RMSPE = sqrt(sspe/n_targets))
 * Errors: EINVAL (bad params / role / config index), ESTATE, ENUMERIC (sspe = NaN),
 * ECUDA, ENOMEM, ENCCL. */
int pgpcv_predict(pgpcv_ctx *ctx, const pgpcv_param *params, int32_t n_params,
                  const int32_t *subset_config, int32_t target_role, double *yhat,
                  double *subset_sspe, double *sspe);

/* Row f4: GLS estimate of a linear mean (Conclusion, Eq. GLS)
 *   beta_hat = (X^T M^{-1} X)^{-1} X^T M^{-1} y,  M = Sigma + lambda I,
 * with M^{-1} X obtained "by a spatial prediction operation" per subset: the
 * rows of M^{-1} [X | y] at a training point are those of the system of the subset whose
 * core holds the point (R23) -- exact when one subset holds all data.  One
 * factorization per subset serves all p + 1 right-hand sides (bordered rows).
 *   X: host double[n * p], row-major per input point (the n points of the partition call,
 *      in their order); only the training points' rows are used.  1 <= p <= 8.  X is
 *      not validated: non-finite entries make the affected sums and beta NaN.
 *   param: one configuration (range, sigma2, nugget).
 *   beta: host double[p] out.  xtmx: double[p*p] row-major or NULL; xtmy: double[p] or NULL
 *      (the summed normal equations X^T M^{-1} X, X^T M^{-1} y).
 * Errors: EINVAL, ESTATE, ENUMERIC (a non-PD subset -> NaN sums; or a singular p x p
 * system -> beta NaN), ECUDA, ENOMEM, ENCCL. */
int pgpcv_gls(pgpcv_ctx *ctx, const double *X, int32_t p, pgpcv_param param, double *beta,
              double *xtmx, double *xtmy);

/* CSR lists of the test points (role 2) per core tile: test_off int64[N+1], test_idx
 * int32[n_test] (ascending point index within a subset).  Either may be NULL.
 * Errors: ESTATE, ECUDA. */
int pgpcv_partition_export_test(pgpcv_ctx *ctx, int64_t *test_off, int32_t *test_idx);

/* Timing and work counts of the last successful pgpcv_cv_loss / pgpcv_evaluate /
 * pgpcv_predict on ctx. */
int pgpcv_last_timing(const pgpcv_ctx *ctx, pgpcv_timing *out);

/* Host-only helper (no GPU needed): LPT assignment of n_items with costs cost[] to
 * `world` owners -- items in descending cost (ties: ascending index), each to the
 * currently least-loaded owner (ties: lowest rank).  owner: int32[n_items] out.
 * This is the rule every evaluation applies after pgpcv_shard, over the subsets it
 * factors in ascending subset id (CV: subsets with validation data; with the likelihood:
 * every subset; predict: subsets with targets; GLS: subsets with training data), cost k^3. */
int pgpcv_lpt_assign(int64_t n_items, const double *cost, int32_t world, int32_t *owner);

/* Diagnostic (no part of the method's data path): evaluate one of the kernel's elementary
 * FP64 functions on n host values x -> y (caller-owned host arrays), on the ctx device with
 * the exact device code the CV kernel inlines, so their accuracy can be tested directly.
 *   fn = PGPCV_MATH_EXP_NEG: exp(x) for x <= 0 (the covariance exp(-d/range));
 *        PGPCV_MATH_SQRT:    sqrt(x) for x >= 0 (the distance of squared offsets);
 *        PGPCV_MATH_RSQRT:   1/sqrt(x) for x > 0 (the Cholesky pivots).
 * Errors: EINVAL (bad fn, n < 0, NULL), ECUDA, ENOMEM. */
#define PGPCV_MATH_EXP_NEG 0
#define PGPCV_MATH_SQRT 1
#define PGPCV_MATH_RSQRT 2
int pgpcv_device_math(pgpcv_ctx *ctx, int32_t fn, int64_t n, const double *x, double *y);

#ifdef __cplusplus
}
#endif

#endif /* PGPCV_H */
