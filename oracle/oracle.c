/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the parallel-CV loss.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_1912_13132_b200/,
 * include/, the CUDA library) may include, link, load or call this file.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs use it.  It shares no code, header, table or constant with the CUDA path.
 *
 * Compiled with:  gcc -O2 -ffp-contract=off -fPIC -shared  (IEEE round-to-nearest,
 * no FMA contraction, SSE2 double arithmetic -- no x87 extended precision except in
 * the explicitly long-double adjudication variant).
 *
 * What it computes (citations: P:n = /root/reference/PAPER.md line n; DESIGN.md
 * "Readings" R1..R18 for every place the paper is silent):
 *
 *   Eq.7:  CV~(y_T, y_V, zeta) = sum_{i=1..N} CV(y~^i_T, y^i_V, zeta)
 *   Eq.4:  CV(y_T, y_V, zeta)  = sum_i (yhat_V[i] - y_V[i])^2
 *   Eq.3:  yhat_p = Sigma_p^T (Sigma + lambda I)^{-1} y,  lambda = tau / sigma^2
 *   Sec.3: c(s1, s2, theta) = exp(-||s1 - s2|| / theta)
 *   Shell: y~^i_T = training data in D_i union D_i^shell (width delta)
 *   Alg.1: create subsets once, per subset local SSPE z_i, combine z = sum z_i
 *
 * Steps follow the algorithm in the paper's order with no blocking, fusion or
 * reordering: brute-force membership, unblocked Cholesky-Banachiewicz, forward then
 * backward substitution, prediction, squared error, fixed ascending sums.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL (-2)
#define OR_ENUMERIC (-3)
#define OR_ENOMEM (-6)

/* ---------------------------------------------------------------------------
 * Partition (Alg.1 lines 2-3; shells P:154-159; readings R1-R6).
 * ------------------------------------------------------------------------- */

/* Tile edges of one axis [a, b) split into K equal tiles (reading R4):
 *   w = (b - a) / K ; e_i = a + i*w (separate multiply and add) ; e_K = b exactly.
 * Returns OR_EINVAL when the edges are not strictly increasing. */
int oracle_edges(double a, double b, int32_t K, double *e) {
    if (!(K >= 1) || !(a < b)) return OR_EINVAL;
    double w = (b - a) / (double)K;
    for (int32_t i = 0; i < K; ++i) {
        double iw = (double)i * w;
        e[i] = a + iw;
    }
    e[K] = b;
    for (int32_t i = 0; i < K; ++i)
        if (!(e[i] < e[i + 1])) return OR_EINVAL;
    return OR_OK;
}

/* Core tile along one axis (reading R3): the unique i with e_i <= x < e_{i+1}, or
 * K-1 when x == e_K (closed domain top).  Brute-force scan of all K intervals. */
static int32_t core_index(double x, const double *e, int32_t K) {
    int32_t found = -1;
    for (int32_t i = 0; i < K; ++i)
        if (e[i] <= x && x < e[i + 1]) found = i;
    if (found < 0 && x == e[K]) found = K - 1;
    return found;
}

/* Dilated-tile membership along one axis (reading R2/R3): lo_i = e_i - delta,
 * hi_i = e_{i+1} + delta, member iff lo_i <= x < hi_i, with hi_{K-1} = +inf. */
static int in_dilated(double x, const double *e, int32_t K, int32_t i, double delta) {
    double lo = e[i] - delta;
    double hi = e[i + 1] + delta;
    if (i == K - 1) hi = INFINITY;
    return lo <= x && x < hi;
}

static int check_inputs(int64_t n, const double *x, const double *y, const uint8_t *role,
                        double xmin, double xmax, double ymin, double ymax,
                        int32_t kx, int32_t ky, double delta) {
    if (n < 0 || kx < 1 || ky < 1 || !(delta >= 0.0) || isinf(delta)) return OR_EINVAL;
    if (!(xmin < xmax) || !(ymin < ymax) || !isfinite(xmin) || !isfinite(xmax) || !isfinite(ymin) ||
        !isfinite(ymax))
        return OR_EINVAL;
    for (int64_t p = 0; p < n; ++p) {
        if (!isfinite(x[p]) || !isfinite(y[p])) return OR_EINVAL;
        if (x[p] < xmin || x[p] > xmax || y[p] < ymin || y[p] > ymax) return OR_EINVAL;
        if (role[p] > 2) return OR_EINVAL;
    }
    return OR_OK;
}

/* Pass 1: per-subset counts.  Subset id s = iy*kx + ix (reading R5).
 * train(s) = {p : role 0, p in the dilated tile s};  val(s) = {p : role core_role,
 * core(p) = s} -- core_role 1 gives the validation lists (reading R6: validation never
 * comes from the shell; Eq.7 writes y^i_V), core_role 2 the test lists predicted
 * with the chosen parameters. */
int oracle_partition_count(int64_t n, const double *x, const double *y, const uint8_t *role,
                           double xmin, double xmax, double ymin, double ymax,
                           int32_t kx, int32_t ky, double delta, uint8_t core_role,
                           int64_t *train_cnt, int64_t *val_cnt) {
    int rc = check_inputs(n, x, y, role, xmin, xmax, ymin, ymax, kx, ky, delta);
    if (rc) return rc;
    double *ex = malloc(sizeof(double) * (kx + 1)), *ey = malloc(sizeof(double) * (ky + 1));
    if (!ex || !ey) { free(ex); free(ey); return OR_ENOMEM; }
    rc = oracle_edges(xmin, xmax, kx, ex);
    if (!rc) rc = oracle_edges(ymin, ymax, ky, ey);
    if (rc) { free(ex); free(ey); return rc; }
    int64_t N = (int64_t)kx * ky;
    for (int64_t s = 0; s < N; ++s) { train_cnt[s] = 0; val_cnt[s] = 0; }
    for (int64_t p = 0; p < n; ++p) {
        if (role[p] == core_role) {
            int32_t ix = core_index(x[p], ex, kx), iy = core_index(y[p], ey, ky);
            val_cnt[(int64_t)iy * kx + ix] += 1;
        } else if (role[p] == 0) {
            for (int32_t iy = 0; iy < ky; ++iy) {
                if (!in_dilated(y[p], ey, ky, iy, delta)) continue;
                for (int32_t ix = 0; ix < kx; ++ix)
                    if (in_dilated(x[p], ex, kx, ix, delta)) train_cnt[(int64_t)iy * kx + ix] += 1;
            }
        }
    }
    free(ex); free(ey);
    return OR_OK;
}

/* Pass 2: fill CSR lists.  Points are visited in ascending index and appended, so
 * each list is in ascending original index (reading R5).  train_off/val_off are the
 * exclusive prefix sums of the pass-1 counts (N+1 entries, computed by the caller). */
int oracle_partition_fill(int64_t n, const double *x, const double *y, const uint8_t *role,
                          double xmin, double xmax, double ymin, double ymax,
                          int32_t kx, int32_t ky, double delta, uint8_t core_role,
                          const int64_t *train_off, int32_t *train_idx,
                          const int64_t *val_off, int32_t *val_idx) {
    int rc = check_inputs(n, x, y, role, xmin, xmax, ymin, ymax, kx, ky, delta);
    if (rc) return rc;
    double *ex = malloc(sizeof(double) * (kx + 1)), *ey = malloc(sizeof(double) * (ky + 1));
    int64_t N = (int64_t)kx * ky;
    int64_t *tpos = malloc(sizeof(int64_t) * N), *vpos = malloc(sizeof(int64_t) * N);
    if (!ex || !ey || !tpos || !vpos) { free(ex); free(ey); free(tpos); free(vpos); return OR_ENOMEM; }
    rc = oracle_edges(xmin, xmax, kx, ex);
    if (!rc) rc = oracle_edges(ymin, ymax, ky, ey);
    if (rc) { free(ex); free(ey); free(tpos); free(vpos); return rc; }
    for (int64_t s = 0; s < N; ++s) { tpos[s] = train_off[s]; vpos[s] = val_off[s]; }
    for (int64_t p = 0; p < n; ++p) {
        if (role[p] == core_role) {
            int32_t ix = core_index(x[p], ex, kx), iy = core_index(y[p], ey, ky);
            int64_t s = (int64_t)iy * kx + ix;
            val_idx[vpos[s]++] = (int32_t)p;
        } else if (role[p] == 0) {
            for (int32_t iy = 0; iy < ky; ++iy) {
                if (!in_dilated(y[p], ey, ky, iy, delta)) continue;
                for (int32_t ix = 0; ix < kx; ++ix)
                    if (in_dilated(x[p], ex, kx, ix, delta)) {
                        int64_t s = (int64_t)iy * kx + ix;
                        train_idx[tpos[s]++] = (int32_t)p;
                    }
            }
        }
    }
    free(ex); free(ey); free(tpos); free(vpos);
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Per-subset CV loss, Eq.4 with Eq.3's predictor, for one (subset, config).
 * Written once as a macro over the real type: `double` is the oracle, `long double`
 * (x87 80-bit) is the adjudication variant for conditioning questions (reading R18).
 * ------------------------------------------------------------------------- */
#define DEFINE_SUBSET_CV(NAME, REAL, EXP, SQRT)                                                    \
int NAME(int64_t k, const double *tx, const double *ty, const double *tv,                          \
         int64_t m, const double *vx, const double *vy, const double *vv,                          \
         double range, double sigma2, double nugget, double *loss_out, double *yhat_out) {         \
    if (!(range > 0) || !(sigma2 > 0) || !(nugget >= 0) || isinf(range) || isinf(sigma2) ||        \
        isinf(nugget))                                                                             \
        return OR_EINVAL;                                                                          \
    /* reading R10: empty validation -> loss exactly 0 */                                          \
    if (m == 0) { *loss_out = 0.0; return OR_OK; }                                                 \
    REAL theta = (REAL)range;                                                                      \
    REAL lambda = (REAL)nugget / (REAL)sigma2; /* P:109 */                                         \
    REAL *L = NULL, *z = NULL, *alpha = NULL;                                                      \
    if (k > 0) {                                                                                   \
        L = (REAL *)malloc(sizeof(REAL) * (size_t)k * (size_t)k);                                  \
        z = (REAL *)malloc(sizeof(REAL) * (size_t)k);                                              \
        alpha = (REAL *)malloc(sizeof(REAL) * (size_t)k);                                          \
        if (!L || !z || !alpha) { free(L); free(z); free(alpha); return OR_ENOMEM; }               \
        /* Sigma + lambda I (Eq.3 second line), lower triangle, row-major. */               \
        for (int64_t i = 0; i < k; ++i) {                                                          \
            for (int64_t j = 0; j < i; ++j) {                                                      \
                REAL dx = (REAL)tx[i] - (REAL)tx[j];                                               \
                REAL dy = (REAL)ty[i] - (REAL)ty[j];                                               \
                REAL d = SQRT(dx * dx + dy * dy);                                                  \
                L[i * k + j] = EXP(-d / theta); /* P:258 */                                        \
            }                                                                                      \
            L[i * k + i] = (REAL)1 + lambda; /* exp(0) = 1 exactly */                              \
        }                                                                                          \
        /* Cholesky-Banachiewicz, row by row, in place on the lower triangle. */                   \
        for (int64_t i = 0; i < k; ++i) {                                                          \
            for (int64_t j = 0; j <= i; ++j) {                                                     \
                REAL s = L[i * k + j];                                                             \
                for (int64_t p = 0; p < j; ++p) s -= L[i * k + p] * L[j * k + p];                  \
                if (i == j) {                                                                      \
                    if (!(s > 0)) { free(L); free(z); free(alpha); return OR_ENUMERIC; }           \
                    L[i * k + i] = SQRT(s);                                                        \
                } else {                                                                           \
                    L[i * k + j] = s / L[j * k + j];                                               \
                }                                                                                  \
            }                                                                                      \
        }                                                                                          \
        /* forward substitution L z = y_T */                                                       \
        for (int64_t i = 0; i < k; ++i) {                                                          \
            REAL s = (REAL)tv[i];                                                                  \
            for (int64_t p = 0; p < i; ++p) s -= L[i * k + p] * z[p];                              \
            z[i] = s / L[i * k + i];                                                               \
        }                                                                                          \
        /* backward substitution L^T alpha = z */                                                  \
        for (int64_t i = k - 1; i >= 0; --i) {                                                     \
            REAL s = z[i];                                                                         \
            for (int64_t p = i + 1; p < k; ++p) s -= L[p * k + i] * alpha[p];                      \
            alpha[i] = s / L[i * k + i];                                                           \
        }                                                                                          \
    }                                                                                              \
    /* prediction yhat_v = sum_j c(v, t_j) alpha_j (Eq.3), squared error (Eq.4) */                 \
    REAL loss = 0;                                                                                 \
    for (int64_t v = 0; v < m; ++v) {                                                              \
        REAL yhat = 0; /* reading R11: k = 0 -> zero-mean prior, yhat = 0 */                       \
        for (int64_t j = 0; j < k; ++j) {                                                          \
            REAL dx = (REAL)vx[v] - (REAL)tx[j];                                                   \
            REAL dy = (REAL)vy[v] - (REAL)ty[j];                                                   \
            REAL d = SQRT(dx * dx + dy * dy);                                                      \
            yhat += EXP(-d / theta) * alpha[j];                                                    \
        }                                                                                          \
        if (yhat_out) yhat_out[v] = (double)yhat;                                                  \
        REAL e = yhat - (REAL)vv[v];                                                               \
        loss += e * e;                                                                             \
    }                                                                                              \
    free(L); free(z); free(alpha);                                                                 \
    *loss_out = (double)loss;                                                                      \
    return OR_OK;                                                                                  \
}

DEFINE_SUBSET_CV(oracle_subset_cv, double, exp, sqrt)
DEFINE_SUBSET_CV(oracle_subset_cv_ld, long double, expl, sqrtl)

/* ---------------------------------------------------------------------------
 * f3 (NEXT): -2 log-likelihood of Eq.2 for one subset's training data,
 *   n log(2 pi) + log det(sigma2 Sigma + tau I) + y^T (sigma2 Sigma + tau I)^{-1} y,
 * evaluated as written: form sigma2*Sigma + tau*I, Cholesky, log det = 2 sum log L_ii,
 * quadratic form = ||L^{-1} y||^2.
 * ------------------------------------------------------------------------- */
int oracle_neg2loglik(int64_t k, const double *tx, const double *ty, const double *tv,
                      double range, double sigma2, double nugget, double *out) {
    if (!(range > 0) || !(sigma2 > 0) || !(nugget >= 0)) return OR_EINVAL;
    if (k == 0) { *out = 0.0; return OR_OK; }
    double *L = malloc(sizeof(double) * (size_t)k * (size_t)k);
    double *z = malloc(sizeof(double) * (size_t)k);
    if (!L || !z) { free(L); free(z); return OR_ENOMEM; }
    for (int64_t i = 0; i < k; ++i) {
        for (int64_t j = 0; j < i; ++j) {
            double dx = tx[i] - tx[j], dy = ty[i] - ty[j];
            double d = sqrt(dx * dx + dy * dy);
            L[i * k + j] = sigma2 * exp(-d / range);
        }
        L[i * k + i] = sigma2 + nugget;
    }
    for (int64_t i = 0; i < k; ++i)
        for (int64_t j = 0; j <= i; ++j) {
            double s = L[i * k + j];
            for (int64_t p = 0; p < j; ++p) s -= L[i * k + p] * L[j * k + p];
            if (i == j) {
                if (!(s > 0)) { free(L); free(z); return OR_ENUMERIC; }
                L[i * k + i] = sqrt(s);
            } else {
                L[i * k + j] = s / L[j * k + j];
            }
        }
    double logdet = 0, quad = 0;
    for (int64_t i = 0; i < k; ++i) {
        double s = tv[i];
        for (int64_t p = 0; p < i; ++p) s -= L[i * k + p] * z[p];
        z[i] = s / L[i * k + i];
        logdet += log(L[i * k + i]);
        quad += z[i] * z[i];
    }
    *out = (double)k * log(2.0 * 3.14159265358979323846) + 2.0 * logdet + quad;
    free(L); free(z);
    return OR_OK;
}
