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

/* ---------------------------------------------------------------------------
 * Row f2: recursive shell-balanced bisection (Fig. "split" right)
 * and the shell cap of P:418-420.  Readings (R19-R23):
 *   - a node is a rectangle [x0,x1) x [y0,y1), closed at the domain's top edges (R3);
 *   - depth d splits along x (a vertical line) when d is even, along y when d is odd
 *     ("the division lines alternate"; SPEC: depth 1 = vertical line);
 *   - counted data: training and validation points (role 0 or 1), never test points;
 *   - "both rectangles together with their shells contain a similar amount of data"
 *     (P:247): a child's count is the number of counted points in its L-inf dilation by
 *     delta (R2/R3 membership: lo <= u < hi, hi = +inf at the domain top);
 *   - candidate split lines: c = 0.5 * (u_j + u_{j+1}) for consecutive distinct values
 *     u_j < u_{j+1} of the split coordinate of counted points in the node's core; the
 *     one minimising |count_left - count_right| wins, ties to the smallest c (SPEC
 *     recursive_partition); no candidate -> c = 0.5 * (x0 + x1) (R21);
 *   - leaves are numbered in heap order: node 1 = D, children of node i are 2i (lower
 *     coordinates) and 2i+1; subset s = leaf id - 2^depth.
 * Plain: every count comes from scanning all n points; the candidates and band are sorted
 * (qsort) and counted with a written-out lower bound.
 * ------------------------------------------------------------------------- */

static int in_dil(double u, double lo, double hi, double top, double delta) {
    double l = lo - delta;
    double h = (hi == top) ? INFINITY : hi + delta;
    return l <= u && u < h;
}
static int in_core(double u, double lo, double hi, double top) {
    return lo <= u && (u < hi || (hi == top && u == top));
}
static int cmp_double(const void *a, const void *b) {
    double x = *(const double *)a, y = *(const double *)b;
    return (x > y) - (x < y);
}
/* number of entries of the sorted array a[0..len) that are < v */
static int64_t count_below(const double *a, int64_t len, double v) {
    int64_t lo = 0, hi = len;
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (a[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* rects: [2^depth * 4] (x0, x1, y0, y1) per leaf; splits: [2^depth] split coordinate of
 * node id (index id, id = 1 .. 2^depth - 1; entry 0 unused). */
int oracle_bisect(int64_t n, const double *x, const double *y, const uint8_t *role,
                  double xmin, double xmax, double ymin, double ymax, int32_t depth, double delta,
                  double *rects, double *splits) {
    if (depth < 0 || depth > 20 || !(delta >= 0.0) || isinf(delta)) return OR_EINVAL;
    int rc = check_inputs(n, x, y, role, xmin, xmax, ymin, ymax, 1, 1, delta);
    if (rc) return rc;
    int64_t nodes = (int64_t)1 << (depth + 1);
    double *R = malloc(sizeof(double) * 4 * (size_t)nodes); /* rect of node id */
    double *band = malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double *core = malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    if (!R || !band || !core) { free(R); free(band); free(core); return OR_ENOMEM; }
    R[4] = xmin; R[5] = xmax; R[6] = ymin; R[7] = ymax;
    for (int32_t d = 0; d < depth; ++d) {
        int axis = d & 1; /* 0: split x, 1: split y */
        for (int64_t id = (int64_t)1 << d; id < ((int64_t)1 << (d + 1)); ++id) {
            const double *r = R + 4 * id;
            int64_t nb = 0, nc = 0;
            for (int64_t p = 0; p < n; ++p) {
                if (role[p] > 1) continue;
                int dx = in_dil(x[p], r[0], r[1], xmax, delta), dy = in_dil(y[p], r[2], r[3], ymax, delta);
                if (dx && dy) band[nb++] = axis ? y[p] : x[p];
                if (in_core(x[p], r[0], r[1], xmax) && in_core(y[p], r[2], r[3], ymax))
                    core[nc++] = axis ? y[p] : x[p];
            }
            qsort(band, (size_t)nb, sizeof(double), cmp_double);
            qsort(core, (size_t)nc, sizeof(double), cmp_double);
            double best_c = 0.5 * (r[2 * axis] + r[2 * axis + 1]);
            int64_t best_score = -1;
            for (int64_t j = 0; j + 1 < nc; ++j) {
                if (!(core[j] < core[j + 1])) continue;
                double c = 0.5 * (core[j] + core[j + 1]);
                int64_t left = count_below(band, nb, c + delta);        /* u <  c + delta */
                int64_t right = nb - count_below(band, nb, c - delta);  /* u >= c - delta */
                int64_t score = left > right ? left - right : right - left;
                if (best_score < 0 || score < best_score) { best_score = score; best_c = c; }
            }
            splits[id] = best_c;
            double *lc = R + 4 * (2 * id), *rc2 = R + 4 * (2 * id + 1);
            for (int i = 0; i < 4; ++i) { lc[i] = r[i]; rc2[i] = r[i]; }
            lc[2 * axis + 1] = best_c; /* left/lower child ends at c */
            rc2[2 * axis] = best_c;    /* right/upper child starts at c */
        }
    }
    for (int64_t s = 0; s < ((int64_t)1 << depth); ++s)
        for (int i = 0; i < 4; ++i) rects[4 * s + i] = R[4 * (((int64_t)1 << depth) + s) + i];
    if (depth == 0) splits[0] = 0.0;
    free(R); free(band); free(core);
    return OR_OK;
}

/* Membership for an arbitrary list of N leaf rectangles (brute force over all rects):
 * train(s) = role 0 in the dilation of rect s; core(s) = role core_role in rect s. */
int oracle_partition_rects_count(int64_t n, const double *x, const double *y, const uint8_t *role,
                                 double xmax, double ymax, int64_t N, const double *rects,
                                 double delta, uint8_t core_role, int64_t *train_cnt, int64_t *val_cnt) {
    for (int64_t s = 0; s < N; ++s) { train_cnt[s] = 0; val_cnt[s] = 0; }
    for (int64_t p = 0; p < n; ++p)
        for (int64_t s = 0; s < N; ++s) {
            const double *r = rects + 4 * s;
            if (role[p] == 0 && in_dil(x[p], r[0], r[1], xmax, delta) && in_dil(y[p], r[2], r[3], ymax, delta))
                train_cnt[s] += 1;
            if (role[p] == core_role && in_core(x[p], r[0], r[1], xmax) && in_core(y[p], r[2], r[3], ymax))
                val_cnt[s] += 1;
        }
    return OR_OK;
}

int oracle_partition_rects_fill(int64_t n, const double *x, const double *y, const uint8_t *role,
                                double xmax, double ymax, int64_t N, const double *rects, double delta,
                                uint8_t core_role, const int64_t *train_off, int32_t *train_idx,
                                const int64_t *val_off, int32_t *val_idx) {
    int64_t *tpos = malloc(sizeof(int64_t) * (size_t)(N > 0 ? N : 1));
    int64_t *vpos = malloc(sizeof(int64_t) * (size_t)(N > 0 ? N : 1));
    if (!tpos || !vpos) { free(tpos); free(vpos); return OR_ENOMEM; }
    for (int64_t s = 0; s < N; ++s) { tpos[s] = train_off[s]; vpos[s] = val_off[s]; }
    for (int64_t p = 0; p < n; ++p) /* ascending p: every list ends up in ascending index */
        for (int64_t s = 0; s < N; ++s) {
            const double *r = rects + 4 * s;
            if (role[p] == 0 && in_dil(x[p], r[0], r[1], xmax, delta) && in_dil(y[p], r[2], r[3], ymax, delta))
                train_idx[tpos[s]++] = (int32_t)p;
            if (role[p] == core_role && in_core(x[p], r[0], r[1], xmax) && in_core(y[p], r[2], r[3], ymax))
                val_idx[vpos[s]++] = (int32_t)p;
        }
    free(tpos); free(vpos);
    return OR_OK;
}

/* SplitMix64 (Steele, Lea & Flood 2014): output i >= 1 of the generator seeded with
 * `seed` is mix(seed + i * 0x9e3779b97f4a7c15). */
uint64_t oracle_splitmix64(uint64_t seed, uint64_t i) {
    uint64_t z = seed + i * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

/* Shell cap (shells with more than 2,000 residuals are reduced "to 2,000 by
 * random sampling"; reading R22): of subset s's training list (ascending p) the shell
 * members -- those outside the core rect -- are sorted by (key, p) with
 * key = splitmix64(seed, s * 2^32 + p + 1) and only the first `cap` are kept; core members
 * are always kept.  Writes the kept list (ascending p) to out, its length to *k_out. */
typedef struct { uint64_t key; int32_t p; } keyed_t;
static int cmp_keyed(const void *a, const void *b) {
    const keyed_t *u = (const keyed_t *)a, *v = (const keyed_t *)b;
    if (u->key != v->key) return u->key < v->key ? -1 : 1;
    return (u->p > v->p) - (u->p < v->p);
}
int oracle_cap_shell(int64_t k, const int32_t *idx, const double *x, const double *y, const double *rect,
                     double xmax, double ymax, int64_t cap, uint64_t seed, int64_t s, int32_t *out,
                     int64_t *k_out) {
    keyed_t *sh = malloc(sizeof(keyed_t) * (size_t)(k > 0 ? k : 1));
    uint8_t *keep = malloc((size_t)(k > 0 ? k : 1));
    if (!sh || !keep) { free(sh); free(keep); return OR_ENOMEM; }
    int64_t nshell = 0;
    for (int64_t i = 0; i < k; ++i) {
        int32_t p = idx[i];
        int core = in_core(x[p], rect[0], rect[1], xmax) && in_core(y[p], rect[2], rect[3], ymax);
        keep[i] = 1;
        if (!core) {
            sh[nshell].key = oracle_splitmix64(seed, ((uint64_t)s << 32) + (uint64_t)p + 1);
            sh[nshell].p = p;
            ++nshell;
        }
    }
    if (nshell > cap) {
        qsort(sh, (size_t)nshell, sizeof(keyed_t), cmp_keyed);
        /* drop the shell members of rank >= cap (lists are ascending in p: find by scan) */
        for (int64_t r = cap; r < nshell; ++r)
            for (int64_t i = 0; i < k; ++i)
                if (idx[i] == sh[r].p) { keep[i] = 0; break; }
    }
    int64_t o = 0;
    for (int64_t i = 0; i < k; ++i)
        if (keep[i]) out[o++] = idx[i];
    *k_out = o;
    free(sh); free(keep);
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Row f4: GLS mean estimation (Conclusion, Eq. GLS):
 *   beta_hat = (X^T M^{-1} X)^{-1} X^T M^{-1} y,  M = Sigma + lambda I.
 * The paper computes M^{-1} X "by a spatial prediction operation on the columns of X"
 * (M^{-1} = (1/lambda)(I - H)).  Parallel reading (R23): as the CV
 * loss replaces the global prediction by subset predictions, the rows of M^{-1} X and
 * M^{-1} y at a training point p are taken from the system of the subset whose CORE holds
 * p, (M^{-1} X)_p ~ (M_s^{-1} X^s)_p; every training point lies in exactly one core, so
 *   X^T M^{-1} X ~ sum_s sum_{p in core_s} X_p^T (M_s^{-1} X^s)_p,  likewise X^T M^{-1} y,
 * exact when one subset holds all data.  This function returns one subset's two partial
 * sums, computed as written: form M_s, Cholesky, solve M_s W = [y | X] column by column
 * (forward then backward substitution), accumulate over the core rows in ascending order.
 *   Xs: k x p row-major covariates of the subset's training points; core[i] = 1 if
 *   training point i lies in the subset's core.  out_A: p x p row-major,
 *   A[a][b] = sum_core X[i][a] W_b[i];  out_b: p, b[a] = sum_core X[i][a] W_y[i].
 * ------------------------------------------------------------------------- */
int oracle_gls_subset(int64_t k, const double *tx, const double *ty, const double *tv, const double *Xs,
                      const uint8_t *core, int32_t p, double range, double sigma2, double nugget,
                      double *out_A, double *out_b) {
    if (!(range > 0) || !(sigma2 > 0) || !(nugget >= 0) || p < 1) return OR_EINVAL;
    for (int32_t a = 0; a < p; ++a) {
        out_b[a] = 0.0;
        for (int32_t b = 0; b < p; ++b) out_A[a * p + b] = 0.0;
    }
    if (k == 0) return OR_OK;
    double lambda = nugget / sigma2;
    double *L = malloc(sizeof(double) * (size_t)k * (size_t)k);
    double *z = malloc(sizeof(double) * (size_t)k);
    double *w = malloc(sizeof(double) * (size_t)k);
    if (!L || !z || !w) { free(L); free(z); free(w); return OR_ENOMEM; }
    for (int64_t i = 0; i < k; ++i) {
        for (int64_t j = 0; j < i; ++j) {
            double dx = tx[i] - tx[j], dy = ty[i] - ty[j];
            L[i * k + j] = exp(-sqrt(dx * dx + dy * dy) / range);
        }
        L[i * k + i] = 1.0 + lambda;
    }
    for (int64_t i = 0; i < k; ++i)
        for (int64_t j = 0; j <= i; ++j) {
            double s = L[i * k + j];
            for (int64_t q = 0; q < j; ++q) s -= L[i * k + q] * L[j * k + q];
            if (i == j) {
                if (!(s > 0)) { free(L); free(z); free(w); return OR_ENUMERIC; }
                L[i * k + i] = sqrt(s);
            } else {
                L[i * k + j] = s / L[j * k + j];
            }
        }
    for (int32_t col = -1; col < p; ++col) { /* col -1: y, else X column col */
        for (int64_t i = 0; i < k; ++i) {
            double s = col < 0 ? tv[i] : Xs[i * p + col];
            for (int64_t q = 0; q < i; ++q) s -= L[i * k + q] * z[q];
            z[i] = s / L[i * k + i];
        }
        for (int64_t i = k - 1; i >= 0; --i) {
            double s = z[i];
            for (int64_t q = i + 1; q < k; ++q) s -= L[q * k + i] * w[q];
            w[i] = s / L[i * k + i];
        }
        for (int64_t i = 0; i < k; ++i) {
            if (!core[i]) continue;
            for (int32_t a = 0; a < p; ++a) {
                if (col < 0) out_b[a] += Xs[i * p + a] * w[i];
                else out_A[a * p + col] += Xs[i * p + a] * w[i];
            }
        }
    }
    free(L); free(z); free(w);
    return OR_OK;
}

/* Solve A beta = b (p x p, row-major) by Gaussian elimination with partial pivoting
 * (largest |pivot|, first on ties).  A singular pivot (exactly 0) gives OR_ENUMERIC. */
int oracle_solve_small(int32_t p, const double *A_in, const double *b_in, double *beta) {
    double A[64 * 64], b[64];
    if (p < 1 || p > 64) return OR_EINVAL;
    for (int32_t i = 0; i < p * p; ++i) A[i] = A_in[i];
    for (int32_t i = 0; i < p; ++i) b[i] = b_in[i];
    for (int32_t c = 0; c < p; ++c) {
        int32_t piv = c;
        for (int32_t r = c + 1; r < p; ++r)
            if (fabs(A[r * p + c]) > fabs(A[piv * p + c])) piv = r;
        if (A[piv * p + c] == 0.0) return OR_ENUMERIC;
        if (piv != c) {
            for (int32_t j = 0; j < p; ++j) { double t = A[c * p + j]; A[c * p + j] = A[piv * p + j]; A[piv * p + j] = t; }
            double t = b[c]; b[c] = b[piv]; b[piv] = t;
        }
        for (int32_t r = c + 1; r < p; ++r) {
            double f = A[r * p + c] / A[c * p + c];
            for (int32_t j = c; j < p; ++j) A[r * p + j] -= f * A[c * p + j];
            b[r] -= f * b[c];
        }
    }
    for (int32_t r = p - 1; r >= 0; --r) {
        double s = b[r];
        for (int32_t j = r + 1; j < p; ++j) s -= A[r * p + j] * beta[j];
        beta[r] = s / A[r * p + r];
    }
    return OR_OK;
}
