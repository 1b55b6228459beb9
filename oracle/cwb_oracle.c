/*
 * cwb_oracle.c -- plain fp64 CPU oracle for binned componentwise boosting
 * (arXiv 2110.03513).  TEST INFRASTRUCTURE ONLY (see cwb_oracle.h).
 *
 * Written from PAPER.md alone, step by step in the paper's order, with the
 * plain definition wherever the paper has a faster equivalent.  No blocking,
 * fusion or reordering.  Compiled with -O2 -ffp-contract=off (no FMA
 * contraction, so every product and sum is rounded as written).
 *
 * Parity pins for every function live in tests/test_oracle_*.py.
 */
#include "cwb_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ bins */

/* "n* = sqrt(n)" (Wood), rounded up (reading G1); n^(1/4). */
int orc_n_star(int64_t n, int rule, int fixed) {
    if (n < 1) return ORC_EINVAL;
    if (rule == 2) return fixed >= 2 ? fixed : ORC_EINVAL;
    if (rule == 0) {
        int64_t s = (int64_t)ceil(sqrt((double)n));
        while (s > 1 && (s - 1) * (s - 1) >= n) s--;
        while (s * s < n) s++;
        return s < 2 ? 2 : (int)s;
    }
    if (rule == 1) {
        int64_t s = (int64_t)ceil(pow((double)n, 0.25));
        while (s > 1 && (s - 1) * (s - 1) * (s - 1) * (s - 1) >= n) s--;
        while (s * s * s * s < n) s++;
        return s < 2 ? 2 : (int)s;
    }
    return ORC_EINVAL;
}

/* z_l = min(x) + (l-1)/(n*-1) (max(x) - min(x)), l = 1..n*, evaluated
 * left to right as printed; the last point is forced to max(x) (reading G18).
 * x goes to design point l if x in (z_l - m1, z_l + m2], m = half the
 * distance to the neighbour; the first interval is closed on the left.  A
 * value on a boundary goes to the lower bin (reading G2).  Boundaries are
 * bnd_l = z_l + (z_{l+1} - z_l)/2; idx(x) = smallest l with x <= bnd_l, else
 * the last bin.  Found by binary search over bnd (no arithmetic rounding). */
int orc_build_bins(const double* x, int64_t n, int n_star, double* z, double* bnd, int32_t* idx) {
    if (n < 1 || n_star < 2) return ORC_EINVAL;
    double lo = x[0], hi = x[0];
    for (int64_t i = 0; i < n; i++) {
        if (!isfinite(x[i])) return ORC_ENONFINITE;
        if (x[i] < lo) lo = x[i];
        if (x[i] > hi) hi = x[i];
    }
    if (!(lo < hi)) return ORC_EDEGENERATE;
    for (int l = 0; l < n_star; l++) {
        double t = (double)l / (double)(n_star - 1);
        z[l] = lo + t * (hi - lo);
    }
    z[n_star - 1] = hi;
    for (int l = 0; l < n_star - 1; l++) bnd[l] = z[l] + (z[l + 1] - z[l]) / 2.0;
    for (int64_t i = 0; i < n; i++) {
        int a = 0, b = n_star - 1; /* answer in [a, b]; b = n*-1 means "none" */
        while (a < b) {
            int mid = a + (b - a) / 2;
            if (x[i] <= bnd[mid]) b = mid;
            else a = mid + 1;
        }
        idx[i] = a;
    }
    return ORC_OK;
}

static int cmp_double(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

int64_t orc_count_distinct(const double* x, int64_t n) {
    double* t = (double*)malloc(sizeof(double) * (size_t)n);
    if (!t) return -1;
    memcpy(t, x, sizeof(double) * (size_t)n);
    qsort(t, (size_t)n, sizeof(double), cmp_double);
    int64_t c = n > 0 ? 1 : 0;
    for (int64_t i = 1; i < n; i++) c += t[i] != t[i - 1];  /* -0.0 == +0.0 */
    free(t);
    return c;
}

/* ----------------------------------------------------------------- basis */

/* "20 knots and degree 3" -> 20 inner knots, d = n_knots + degree + 1
 * (reading G5). */
int orc_basis_dim(int degree, int n_knots) { return n_knots + degree + 1; }

/* P:L822 g_k(x) = (B_1(x), ..., B_d(x)): B-splines (P-splines, Eilers & Marx).
 * Knots equidistant over [lo, hi] extended by `degree` knots on each side
 * (reading G6): t_q = lo + (q - degree) h, h = (hi - lo)/(n_knots + 1),
 * q = 0 .. n_knots + 2 degree + 1.  Cox-de Boor recursion:
 *   B_{q,0}(x) = 1{t_q <= x < t_{q+1}}
 *   B_{q,p}(x) = (x - t_q)/(t_{q+p} - t_q) B_{q,p-1}(x)
 *              + (t_{q+p+1} - x)/(t_{q+p+1} - t_{q+1}) B_{q+1,p-1}(x). */
int orc_bspline_basis(const double* x, int64_t m, double lo, double hi, int degree, int n_knots,
                      double* out) {
    if (degree < 0 || n_knots < 0 || !(lo < hi)) return ORC_EINVAL;
    int nk = n_knots + 2 * degree + 2;
    int d = orc_basis_dim(degree, n_knots);
    double* t = (double*)malloc(sizeof(double) * nk);
    double* N = (double*)malloc(sizeof(double) * nk);
    if (!t || !N) { free(t); free(N); return ORC_ENOMEM; }
    double h = (hi - lo) / (double)(n_knots + 1);
    for (int q = 0; q < nk; q++) t[q] = lo + (double)(q - degree) * h;
    for (int64_t i = 0; i < m; i++) {
        double xi = x[i];
        for (int q = 0; q < nk - 1; q++) N[q] = (t[q] <= xi && xi < t[q + 1]) ? 1.0 : 0.0;
        for (int p = 1; p <= degree; p++) {
            for (int q = 0; q < nk - 1 - p; q++) {
                double a = (xi - t[q]) / (t[q + p] - t[q]) * N[q];
                double b = (t[q + p + 1] - xi) / (t[q + p + 1] - t[q + 1]) * N[q + 1];
                N[q] = a + b;
            }
        }
        for (int j = 0; j < d; j++) out[i * d + j] = N[j];
    }
    free(t);
    free(N);
    return ORC_OK;
}

/* Supp. P:L312: D^{1/2}(i) = (0..0, 1, -2, 1, 0..0) in R^{(d-2) x d}; D = D^{1/2 T} D^{1/2}. */
void orc_penalty(int d, double* D) {
    int r = d - 2;
    double* Dl = (double*)calloc((size_t)(r > 0 ? r : 1) * d, sizeof(double));
    for (int i = 0; i < r; i++) {
        Dl[i * d + i] = 1.0;
        Dl[i * d + i + 1] = -2.0;
        Dl[i * d + i + 2] = 1.0;
    }
    for (int a = 0; a < d; a++)
        for (int b = 0; b < d; b++) {
            double s = 0.0;
            for (int i = 0; i < r; i++) s += Dl[i * d + a] * Dl[i * d + b];
            D[a * d + b] = s;
        }
    free(Dl);
}

/* ------------------------------------------------- binned matrix products */

/* Algorithm binMatMat, P:L887-892 (reading G3/G4: w_i is the observation
 * weight; column idx(i) of the d x n* matrix U receives w_i Zb(idx(i))^T). */
void orc_bin_mat_mat(const double* Zb, int n_star, int d, const int32_t* idx, const double* w,
                     int64_t n, double* out) {
    double* U = (double*)calloc((size_t)d * n_star, sizeof(double)); /* U = 0_{d x n*} */
    for (int64_t i = 0; i < n; i++) {
        int l = idx[i];
        double wi = w ? w[i] : 1.0;
        for (int j = 0; j < d; j++) U[j * n_star + l] += wi * Zb[l * d + j];
    }
    for (int a = 0; a < d; a++) /* return U Zb */
        for (int b = 0; b < d; b++) {
            double s = 0.0;
            for (int l = 0; l < n_star; l++) s += U[a * n_star + l] * Zb[l * d + b];
            out[a * d + b] = s;
        }
    free(U);
}

/* Algorithm binMatVec. */
void orc_bin_mat_vec(const double* Zb, int n_star, int d, const int32_t* idx, const double* w,
                     const double* r, int64_t n, double* out) {
    double* u = (double*)calloc((size_t)n_star, sizeof(double)); /* u = 0_{n*} */
    for (int64_t i = 0; i < n; i++) u[idx[i]] += (w ? w[i] : 1.0) * r[i];
    for (int j = 0; j < d; j++) { /* return Zb^T u */
        double s = 0.0;
        for (int l = 0; l < n_star; l++) s += Zb[l * d + j] * u[l];
        out[j] = s;
    }
    free(u);
}

/* Row i of the materialised design matrix: rows[idx[i]] or rows[i]. */
static inline const double* zrow(const double* rows, const int32_t* idx, int d, int64_t i) {
    return rows + (size_t)d * (size_t)(idx ? idx[i] : i);
}

static void dense_ztwz_rows(const double* rows, const int32_t* idx, int d, const double* w,
                            int64_t n, double* out) {
    for (int a = 0; a < d * d; a++) out[a] = 0.0;
    for (int64_t i = 0; i < n; i++) {
        const double* zi = zrow(rows, idx, d, i);
        double wi = w ? w[i] : 1.0;
        for (int a = 0; a < d; a++)
            for (int b = 0; b < d; b++) out[a * d + b] += zi[a] * wi * zi[b];
    }
}

static void dense_ztwr_rows(const double* rows, const int32_t* idx, int d, const double* w,
                            const double* r, int64_t n, double* out) {
    for (int a = 0; a < d; a++) out[a] = 0.0;
    for (int64_t i = 0; i < n; i++) {
        const double* zi = zrow(rows, idx, d, i);
        double wr = (w ? w[i] : 1.0) * r[i];
        for (int a = 0; a < d; a++) out[a] += zi[a] * wr;
    }
}

void orc_dense_ztwz(const double* Zb, int d, const int32_t* idx, const double* w, int64_t n,
                    double* out) {
    dense_ztwz_rows(Zb, idx, d, w, n, out);
}

void orc_dense_ztwr(const double* Zb, int d, const int32_t* idx, const double* w,
                    const double* r, int64_t n, double* out) {
    dense_ztwr_rows(Zb, idx, d, w, r, n, out);
}

/* ------------------------------------------------------- linear algebra */

/* Z^T Z = L L^T. */
int orc_cholesky(const double* A, int d, double* L) {
    for (int a = 0; a < d * d; a++) L[a] = 0.0;
    for (int i = 0; i < d; i++)
        for (int j = 0; j <= i; j++) {
            double s = A[i * d + j];
            for (int q = 0; q < j; q++) s -= L[i * d + q] * L[j * d + q];
            if (i == j) {
                if (!(s > 0.0)) return ORC_EINVAL;
                L[i * d + i] = sqrt(s);
            } else {
                L[i * d + j] = s / L[j * d + j];
            }
        }
    return ORC_OK;
}

/* P:L843 forward/backward solving with the factor. */
static void chol_fb(const double* L, int d, const double* b, double* x) {
    for (int i = 0; i < d; i++) { /* L y = b */
        double s = b[i];
        for (int q = 0; q < i; q++) s -= L[i * d + q] * x[q];
        x[i] = s / L[i * d + i];
    }
    for (int i = d - 1; i >= 0; i--) { /* L^T x = y */
        double s = x[i];
        for (int q = i + 1; q < d; q++) s -= L[q * d + i] * x[q];
        x[i] = s / L[i * d + i];
    }
}

int orc_chol_solve(const double* A, int d, const double* b, double* x) {
    double* L = (double*)malloc(sizeof(double) * d * d);
    int st = orc_cholesky(A, d, L);
    if (st == ORC_OK) chol_fb(L, d, b, x);
    free(L);
    return st;
}

/* ---------------------------------------------------- degrees of freedom */

/* Supp. P:L307-318: H = Z (Z^T W Z + lambda D)^-1 Z^T W (W = I here),
 * df1 = tr H, df2 = tr(2H - H H).  With A = G + lambda D, G = Z^T Z and the
 * cyclic trace identity, tr H = tr(A^-1 G) and tr(H H) = tr(A^-1 G A^-1 G). */
int orc_df(const double* G, const double* D, int d, double lambda, int kind, double* df_out) {
    double* A = (double*)malloc(sizeof(double) * d * d);
    double* L = (double*)malloc(sizeof(double) * d * d);
    double* X = (double*)malloc(sizeof(double) * d * d); /* X = A^-1 G */
    double* col = (double*)malloc(sizeof(double) * d);
    double* sol = (double*)malloc(sizeof(double) * d);
    for (int a = 0; a < d * d; a++) A[a] = G[a] + lambda * D[a];
    int st = orc_cholesky(A, d, L);
    if (st == ORC_OK) {
        for (int c = 0; c < d; c++) {
            for (int r = 0; r < d; r++) col[r] = G[r * d + c];
            chol_fb(L, d, col, sol);
            for (int r = 0; r < d; r++) X[r * d + c] = sol[r];
        }
        double tr = 0.0;
        for (int j = 0; j < d; j++) tr += X[j * d + j];
        if (kind == 2) {
            double tr2 = 0.0;
            for (int a = 0; a < d; a++)
                for (int b = 0; b < d; b++) tr2 += X[a * d + b] * X[b * d + a];
            *df_out = 2.0 * tr - tr2;
        } else {
            *df_out = tr;
        }
    }
    free(A); free(L); free(X); free(col); free(sol);
    return st;
}

/* Supp. P:L316-319: equal df for every learner; "no analytic solution ...
 * must be solved numerically".  df(lambda) is decreasing in lambda: bracket
 * by doubling/halving, then bisect to the resolution of double. */
int orc_df_to_lambda(const double* G, const double* D, int d, double target, int kind,
                     double* lambda_out) {
    if (!(target > 0.0) || target > (double)d) return ORC_ECALIB;
    double v;
    if (d <= 2) {
        /* no second differences (Delta has d - 2 = 0 rows): D = 0 and df(lambda) =
         * rank(Z^T Z) for every lambda -- the target is met by any lambda or by none (the
         * degree-1, no-knot learner of S:L383 with df = 2) */
        if (orc_df(G, D, d, 1.0, kind, &v) != ORC_OK || fabs(v - target) > 1e-9) return ORC_ECALIB;
        *lambda_out = 1.0;
        return ORC_OK;
    }
    double hi = 1.0;
    for (;;) {
        if (orc_df(G, D, d, hi, kind, &v) != ORC_OK) return ORC_ECALIB;
        if (v <= target) break;
        hi *= 2.0;
        if (hi > 1e300) return ORC_ECALIB;
    }
    if (v == target) { *lambda_out = hi; return ORC_OK; }
    double lo = hi / 2.0;
    for (;;) {
        if (lo < 1e-300) return ORC_ECALIB;
        if (orc_df(G, D, d, lo, kind, &v) != ORC_OK) return ORC_ECALIB;
        if (v > target) break;
        hi = lo;
        lo /= 2.0;
    }
    for (int it = 0; it < 400; it++) {
        double mid = lo + (hi - lo) / 2.0;
        if (!(mid > lo && mid < hi)) break;
        if (orc_df(G, D, d, mid, kind, &v) != ORC_OK) return ORC_ECALIB;
        if (v > target) lo = mid;
        else hi = mid;
    }
    *lambda_out = lo + (hi - lo) / 2.0;
    if (orc_df(G, D, d, *lambda_out, kind, &v) != ORC_OK) return ORC_ECALIB;
    if (fabs(v - target) > 1e-9) return ORC_ECALIB;
    return ORC_OK;
}

/* ------------------------------------------------------------------ pool */

void orc_pool_free(orc_pool* p) {
    if (!p) return;
    free(p->lo); free(p->hi); free(p->z); free(p->bnd); free(p->idx); free(p->Zb);
    free(p->Zx); free(p->G); free(p->D); free(p->lambda); free(p->L); free(p->nsk);
    free(p);
}

/* Pool construction ("each base learner that uses binning
 * individually calculates the bin values z, the reduced design matrix Zb and
 * the index vector idx"; P:L846 caching; supp. P:L316-319 df calibration). */
int orc_pool_new(const double* X, int64_t n, int K, const orc_config* cfg, int mode, orc_pool** out) {
    if (K < 1) return ORC_EEMPTY;
    if (n < 2 || !cfg || mode < 0 || mode > 2) return ORC_EINVAL;
    int n_star = orc_n_star(n, cfg->n_star_rule, cfg->n_star_fixed);
    if (n_star < 0) return n_star;
    int d = orc_basis_dim(cfg->degree, cfg->n_knots);
    orc_pool* p = (orc_pool*)calloc(1, sizeof(orc_pool));
    p->K = K; p->n = n; p->n_star = n_star; p->d = d; p->mode = mode;
    p->degree = cfg->degree; p->n_knots = cfg->n_knots;
    p->lo = (double*)malloc(sizeof(double) * K);
    p->hi = (double*)malloc(sizeof(double) * K);
    p->z = (double*)malloc(sizeof(double) * K * n_star);
    p->bnd = (double*)malloc(sizeof(double) * K * (n_star - 1));
    p->idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)K * n);
    p->Zb = (double*)malloc(sizeof(double) * (size_t)K * n_star * d);
    p->G = (double*)malloc(sizeof(double) * K * d * d);
    p->D = (double*)malloc(sizeof(double) * d * d);
    p->lambda = (double*)malloc(sizeof(double) * K);
    p->L = (double*)malloc(sizeof(double) * K * d * d);
    p->nsk = (int32_t*)malloc(sizeof(int32_t) * K);
    if (mode == ORC_MODE_UNBINNED) p->Zx = (double*)malloc(sizeof(double) * (size_t)K * n * d);
    if (!p->lo || !p->hi || !p->z || !p->bnd || !p->idx || !p->Zb || !p->G || !p->D || !p->lambda ||
        !p->L || !p->nsk || (mode == ORC_MODE_UNBINNED && !p->Zx)) {
        orc_pool_free(p);
        return ORC_ENOMEM;
    }
    orc_penalty(d, p->D);
    int st = ORC_OK;
    for (int k = 0; k < K && st == ORC_OK; k++) {
        const double* x = X + (size_t)k * n;
        double* z = p->z + (size_t)k * n_star;
        /* n* clamped to the count of distinct values, per learner;
         * the learner's bins are those of n* = nsk, stored in the first nsk slots */
        const int64_t nd = orc_count_distinct(x, n);
        if (nd < 0) { st = ORC_ENOMEM; break; }
        const int nsk = nd < n_star ? (int)nd : n_star;
        if (nsk < 2) {  /* a constant feature (1 distinct value) */
            for (int64_t i = 0; i < n; i++)
                if (!isfinite(x[i])) { st = ORC_ENONFINITE; break; }
            if (st == ORC_OK) st = ORC_EDEGENERATE;
            break;
        }
        p->nsk[k] = nsk;
        double* bk = p->bnd + (size_t)k * (n_star - 1);
        st = orc_build_bins(x, n, nsk, z, bk, p->idx + (size_t)k * n);
        if (st != ORC_OK) break;
        p->lo[k] = z[0];
        p->hi[k] = z[nsk - 1];
        for (int l = nsk; l < n_star; l++) z[l] = p->hi[k];
        for (int l = nsk - 1; l < n_star - 1; l++) bk[l] = INFINITY;
        double* Zb = p->Zb + (size_t)k * n_star * d;
        st = orc_bspline_basis(z, n_star, p->lo[k], p->hi[k], cfg->degree, cfg->n_knots, Zb);
        if (st != ORC_OK) break;
        double* G = p->G + (size_t)k * d * d;
        if (mode == ORC_MODE_BINNED) {
            orc_bin_mat_mat(Zb, n_star, d, p->idx + (size_t)k * n, NULL, n, G);
        } else if (mode == ORC_MODE_DENSE) {
            dense_ztwz_rows(Zb, p->idx + (size_t)k * n, d, NULL, n, G);
        } else {
            double* Zx = p->Zx + (size_t)k * n * d;
            st = orc_bspline_basis(x, n, p->lo[k], p->hi[k], cfg->degree, cfg->n_knots, Zx);
            if (st != ORC_OK) break;
            dense_ztwz_rows(Zx, NULL, d, NULL, n, G);
        }
        st = orc_df_to_lambda(G, p->D, d, cfg->df, cfg->df_kind, &p->lambda[k]);
        if (st != ORC_OK) break;
        double* A = (double*)malloc(sizeof(double) * d * d);
        for (int a = 0; a < d * d; a++) A[a] = G[a] + p->lambda[k] * p->D[a];
        st = orc_cholesky(A, d, p->L + (size_t)k * d * d);
        free(A);
        if (st != ORC_OK) st = ORC_ECALIB;
    }
    if (st != ORC_OK) { orc_pool_free(p); return st; }
    *out = p;
    return ORC_OK;
}

/* ------------------------------------------------------------ find best */

typedef struct {
    double *s, *theta, *fz, *A;
    double* sse_all;  /* K: SSE of every learner (tie-following mode only) */
} scratch;

static void scratch_init(scratch* w, int d, int n_star) {
    w->s = (double*)malloc(sizeof(double) * d);
    w->theta = (double*)malloc(sizeof(double) * d);
    w->fz = (double*)malloc(sizeof(double) * (n_star > 0 ? n_star : 1));
    w->A = (double*)malloc(sizeof(double) * d * d);
    w->sse_all = NULL;
}

static void scratch_free(scratch* w) { free(w->s); free(w->theta); free(w->fz); free(w->A); free(w->sse_all); }

/* Fit learner k to r (supp. eq. pen-regr): theta = (G + lambda D)^-1 Z^T r,
 * and its SSE = sum_i (r_i - Z(i) theta)^2 (unpenalised, reading G12). */
static double fit_one(const orc_pool* p, int k, const double* r, scratch* w, double* theta) {
    int d = p->d, n_star = p->n_star;
    int64_t n = p->n;
    const int32_t* idx = p->idx + (size_t)k * n;
    const double* Zb = p->Zb + (size_t)k * n_star * d;
    const double* G = p->G + (size_t)k * d * d;
    double sse = 0.0;
    if (p->mode == ORC_MODE_BINNED) {
        orc_bin_mat_vec(Zb, n_star, d, idx, NULL, r, n, w->s); /* P:L915 binMatVec */
        chol_fb(p->L + (size_t)k * d * d, d, w->s, theta);    /* P:L846 cached factor */
        for (int l = 0; l < n_star; l++) {
            double v = 0.0;
            for (int j = 0; j < d; j++) v += Zb[l * d + j] * theta[j];
            w->fz[l] = v;
        }
        for (int64_t i = 0; i < n; i++) {
            double e = r[i] - w->fz[idx[i]];
            sse += e * e;
        }
        return sse;
    }
    const double* rows = (p->mode == ORC_MODE_DENSE) ? Zb : p->Zx + (size_t)k * n * d;
    const int32_t* ridx = (p->mode == ORC_MODE_DENSE) ? idx : NULL;
    dense_ztwr_rows(rows, ridx, d, NULL, r, n, w->s);
    for (int a = 0; a < d * d; a++) w->A[a] = G[a] + p->lambda[k] * p->D[a];
    orc_chol_solve(w->A, d, w->s, theta);
    for (int64_t i = 0; i < n; i++) {
        const double* zi = zrow(rows, ridx, d, i);
        double v = 0.0;
        for (int j = 0; j < d; j++) v += zi[j] * theta[j];
        double e = r[i] - v;
        sse += e * e;
    }
    return sse;
}

static void find_best_ws(const orc_pool* p, const double* r, scratch* w, int32_t* k_out,
                         double* theta_out, double* sse_out, double* sse_all, double* gap_out) {
    int d = p->d;
    int best = -1;
    double best_sse = 0.0, second = INFINITY;
    for (int k = 0; k < p->K; k++) {
        double sse = fit_one(p, k, r, w, w->theta);
        if (sse_all) sse_all[k] = sse;
        if (best < 0 || sse < best_sse) { /* strict: lowest k wins ties */
            if (best >= 0) second = best_sse;
            best = k;
            best_sse = sse;
            for (int j = 0; j < d; j++) theta_out[j] = w->theta[j];
        } else if (sse < second) {
            second = sse;
        }
    }
    *k_out = best;
    *sse_out = best_sse;
    if (gap_out) *gap_out = second - best_sse;
}

int orc_find_best(const orc_pool* p, const double* r, int32_t* k_out, double* theta_out,
                  double* sse_out, double* sse_all_out, double* gap_out) {
    if (!p || p->K < 1) return ORC_EEMPTY;
    for (int64_t i = 0; i < p->n; i++)
        if (!isfinite(r[i])) return ORC_ENONFINITE;
    scratch w;
    scratch_init(&w, p->d, p->n_star);
    find_best_ws(p, r, &w, k_out, theta_out, sse_out, sse_all_out, gap_out);
    scratch_free(&w);
    return ORC_OK;
}

/* ---------------------------------------------------------------- train */

typedef struct {
    const orc_pool* p;
    const double* Y;
    int B, M, tid, nth;
    double nu;
    double *offset, *theta_agg, *sse_trace, *risk_trace, *gap_trace, *f_out;
    int32_t* k_trace;
    int loss; /* ORC_LOSS_L2 or ORC_LOSS_BERNOULLI */
    const int32_t* follow; /* [M][B] learner sequence to follow at verified near-ties (NULL: none) */
    double tie_rtol;
    int32_t* followed;     /* [B] number of iterations at which the followed learner was taken */
} train_job;

/* Bernoulli loss of the logistic model, y in {0, 1}:
 * L(y, f) = log(1 + exp(f)) - y f, written so that exp never overflows. */
static double bern_loss(double y, double f) {
    double sp = f > 0.0 ? f + log1p(exp(-f)) : log1p(exp(f));
    return sp - y * f;
}
/* pseudo residual -dL/df = y - 1 / (1 + exp(-f)) */
static double bern_resid(double y, double f) { return y - 1.0 / (1.0 + exp(-f)); }

/* Alg. 1 supp., one replication at a time. */
static void train_one(const train_job* J, int b, scratch* w, double* f, double* r, double* theta) {
    const orc_pool* p = J->p;
    int64_t n = p->n;
    int d = p->d, K = p->K, B = J->B;
    const double* y = J->Y + (size_t)b * n;
    /* line 2: f0 = argmin_c R_emp(c): mean(y) for L2, log(p / (1 - p)) with p = mean(y) for
     * the Bernoulli loss (S:L319 reading; the caller checked 0 < p < 1) */
    double sy = 0.0;
    for (int64_t i = 0; i < n; i++) sy += y[i];
    double f0 = sy / (double)n;
    if (J->loss == ORC_LOSS_BERNOULLI) f0 = log(f0 / (1.0 - f0));
    J->offset[b] = f0;
    for (int64_t i = 0; i < n; i++) f[i] = f0;
    double* agg = J->theta_agg + (size_t)b * K * d;
    for (int a = 0; a < K * d; a++) agg[a] = 0.0;
    for (int m = 0; m < J->M; m++) {
        /* line 4: pseudo residuals r = -dL/df: y - f for L = 1/2 (y - f)^2 (G9),
         * y - 1 / (1 + exp(-f)) for the Bernoulli loss */
        for (int64_t i = 0; i < n; i++) r[i] = J->loss == ORC_LOSS_BERNOULLI ? bern_resid(y[i], f[i]) : y[i] - f[i];
        /* lines 5-9: fit every learner, SSE, argmin */
        int32_t ks;
        double sse, gap;
        find_best_ws(p, r, w, &ks, theta, &sse, J->follow ? w->sse_all : NULL, &gap);
        if (J->follow) {  /* tie-following: take the given learner when its SSE is
                             within tie_rtol of the minimum -- several results are correct at a near-tie */
            const int32_t kf = J->follow[(size_t)m * B + b];
            if (kf != ks && kf >= 0 && kf < K && w->sse_all[kf] - sse <= J->tie_rtol * fabs(sse)) {
                sse = w->sse_all[kf];
                ks = kf;
                fit_one(p, ks, r, w, theta);
                J->followed[b]++;
            }
        }
        /* line 10: f += nu b_{k*}(x, theta) */
        const double* Zb = p->Zb + (size_t)ks * p->n_star * d;
        const int32_t* idx = p->idx + (size_t)ks * n;
        const double* rows = (p->mode == ORC_MODE_UNBINNED) ? p->Zx + (size_t)ks * n * d : Zb;
        for (int64_t i = 0; i < n; i++) {
            const double* zi = (p->mode == ORC_MODE_UNBINNED) ? rows + (size_t)i * d : Zb + (size_t)idx[i] * d;
            double v = 0.0;
            for (int j = 0; j < d; j++) v += zi[j] * theta[j];
            f[i] = f[i] + J->nu * v;
        }
        /* P:L838 aggregation (with nu, reading G10) */
        for (int j = 0; j < d; j++) agg[ks * d + j] += J->nu * theta[j];
        double rs = 0.0;
        for (int64_t i = 0; i < n; i++) {
            if (J->loss == ORC_LOSS_BERNOULLI) {
                rs += bern_loss(y[i], f[i]);
            } else {
                double e = y[i] - f[i];
                rs += 0.5 * e * e;
            }
        }
        J->k_trace[(size_t)m * B + b] = ks;
        J->sse_trace[(size_t)m * B + b] = sse;
        J->risk_trace[(size_t)m * B + b] = rs / (double)n;
        if (J->gap_trace) J->gap_trace[(size_t)m * B + b] = gap;
    }
    if (J->f_out)
        for (int64_t i = 0; i < n; i++) J->f_out[(size_t)b * n + i] = f[i];
}

static void* train_worker(void* arg) {
    train_job* J = (train_job*)arg;
    int64_t n = J->p->n;
    scratch w;
    scratch_init(&w, J->p->d, J->p->n_star);
    if (J->follow) w.sse_all = (double*)malloc(sizeof(double) * J->p->K);
    double* f = (double*)malloc(sizeof(double) * n);
    double* r = (double*)malloc(sizeof(double) * n);
    double* theta = (double*)malloc(sizeof(double) * J->p->d);
    for (int b = J->tid; b < J->B; b += J->nth) train_one(J, b, &w, f, r, theta);
    free(f); free(r); free(theta);
    scratch_free(&w);
    return NULL;
}

static int train_loss(const orc_pool* p, const double* Y, int B, int loss, double nu, int M, int n_threads,
                      double* offset, double* theta_agg, int32_t* k_trace, double* sse_trace,
                      double* risk_trace, double* gap_trace, double* f_out, const int32_t* follow,
                      double tie_rtol, int32_t* followed);

int orc_train(const orc_pool* p, const double* Y, int B, double nu, int M, int n_threads,
              double* offset, double* theta_agg, int32_t* k_trace, double* sse_trace,
              double* risk_trace, double* gap_trace, double* f_out) {
    return train_loss(p, Y, B, ORC_LOSS_L2, nu, M, n_threads, offset, theta_agg, k_trace, sse_trace, risk_trace,
                      gap_trace, f_out, NULL, 0.0, NULL);
}

int orc_train_follow(const orc_pool* p, const double* Y, int B, double nu, int M, int n_threads,
                     const int32_t* follow, double tie_rtol, double* offset, double* theta_agg, int32_t* k_trace,
                     double* sse_trace, double* risk_trace, double* gap_trace, double* f_out, int32_t* followed) {
    if (!follow || !followed || !(tie_rtol >= 0.0)) return ORC_EINVAL;
    for (int b = 0; b < B; b++) followed[b] = 0;
    return train_loss(p, Y, B, ORC_LOSS_L2, nu, M, n_threads, offset, theta_agg, k_trace, sse_trace, risk_trace,
                      gap_trace, f_out, follow, tie_rtol, followed);
}

int orc_train_loss(const orc_pool* p, const double* Y, int B, int loss, double nu, int M, int n_threads,
                   double* offset, double* theta_agg, int32_t* k_trace, double* sse_trace,
                   double* risk_trace, double* gap_trace, double* f_out) {
    return train_loss(p, Y, B, loss, nu, M, n_threads, offset, theta_agg, k_trace, sse_trace, risk_trace,
                      gap_trace, f_out, NULL, 0.0, NULL);
}

static int train_loss(const orc_pool* p, const double* Y, int B, int loss, double nu, int M, int n_threads,
                      double* offset, double* theta_agg, int32_t* k_trace, double* sse_trace,
                      double* risk_trace, double* gap_trace, double* f_out, const int32_t* follow,
                      double tie_rtol, int32_t* followed) {
    if (!p || p->K < 1) return ORC_EEMPTY;
    if (B < 1 || M < 0 || !(nu >= 0.0) || (loss != ORC_LOSS_L2 && loss != ORC_LOSS_BERNOULLI)) return ORC_EINVAL;
    for (int64_t a = 0; a < (int64_t)B * p->n; a++)
        if (!isfinite(Y[a])) return ORC_ENONFINITE;
    if (loss == ORC_LOSS_BERNOULLI) {  /* y in {0, 1}; mean(y) in (0, 1) */
        for (int64_t a = 0; a < (int64_t)B * p->n; a++)
            if (Y[a] != 0.0 && Y[a] != 1.0) return ORC_EINVAL;
        for (int b = 0; b < B; b++) {
            double sy = 0.0;
            for (int64_t i = 0; i < p->n; i++) sy += Y[(size_t)b * p->n + i];
            if (sy == 0.0 || sy == (double)p->n) return ORC_EDEGENERATE;
        }
    }
    if (n_threads < 1) n_threads = 1;
    if (n_threads > B) n_threads = B;
    train_job* jobs = (train_job*)malloc(sizeof(train_job) * n_threads);
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * n_threads);
    for (int t = 0; t < n_threads; t++) {
        train_job J = {p, Y, B, M, t, n_threads, nu, offset, theta_agg, sse_trace,
                       risk_trace, gap_trace, f_out, k_trace, loss, follow, tie_rtol, followed};
        jobs[t] = J;
    }
    for (int t = 1; t < n_threads; t++) pthread_create(&th[t], NULL, train_worker, &jobs[t]);
    train_worker(&jobs[0]);
    for (int t = 1; t < n_threads; t++) pthread_join(th[t], NULL);
    free(jobs);
    free(th);
    return ORC_OK;
}

/* ------------------------------------------------------------------ ACWB */

typedef struct {
    const orc_pool* p;
    const double* Y;
    int B, M, tid, nth;
    double nu, gamma;
    double *offset, *theta_f, *theta_h, *sse_trace, *sse_cor_trace, *risk_trace, *gap_trace, *gap_cor_trace;
    double *f_out, *h_out;
    int32_t *k_trace, *kcor_trace;
} acwb_job;

/* fitted values of learner k with parameters theta at every row: b_k(x_i, theta) */
static void learner_values(const orc_pool* p, int k, const double* theta, double* out) {
    int d = p->d;
    int64_t n = p->n;
    const double* Zb = p->Zb + (size_t)k * p->n_star * d;
    const int32_t* idx = p->idx + (size_t)k * n;
    for (int64_t i = 0; i < n; i++) {
        const double* zi = (p->mode == ORC_MODE_UNBINNED) ? p->Zx + ((size_t)k * n + i) * d : Zb + (size_t)idx[i] * d;
        double v = 0.0;
        for (int j = 0; j < d; j++) v += zi[j] * theta[j];
        out[i] = v;
    }
}

/* Algorithm 2 (ACWB), one replication, literally: f, h, g, c are the fitted
 * values of the primary, momentum and combined models and the error-corrected pseudo
 * residuals.  Readings: the step of the primary model is nu (the
 * prose's beta); eta_m = gamma nu / theta_m; the correction residual uses
 * the previous iteration's correction learner b_{k_cor^[m-1]}(x, theta_cor^[m-1])
 * (P:L949 prints theta_cor^[m], not yet defined at that point); parameters per P:L966:
 * theta_g = (1 - theta_m) theta_f + theta_m theta_h, theta_f = theta_g + nu e_k theta,
 * theta_h += eta_m e_kcor theta_cor, both starting at zero (the offset is shared). */
static void acwb_one(const acwb_job* J, int b, scratch* w, double* f, double* h, double* g, double* r,
                     double* c, double* bprev, double* bcur, double* theta, double* theta_cor) {
    const orc_pool* p = J->p;
    int64_t n = p->n;
    int d = p->d, K = p->K, B = J->B;
    const double* y = J->Y + (size_t)b * n;
    /* line 2: f0 = argmin_c R_emp(c) = mean(y); h0 = g0 = f0 */
    double sy = 0.0;
    for (int64_t i = 0; i < n; i++) sy += y[i];
    double f0 = sy / (double)n;
    J->offset[b] = f0;
    for (int64_t i = 0; i < n; i++) { f[i] = f0; h[i] = f0; g[i] = f0; }
    double* tf = J->theta_f + (size_t)b * K * d;
    double* th = J->theta_h + (size_t)b * K * d;
    for (int a = 0; a < K * d; a++) { tf[a] = 0.0; th[a] = 0.0; }
    for (int m = 1; m <= J->M; m++) {
        double vt = 2.0 / (double)(m + 1);                                /* line 4 */
        for (int64_t i = 0; i < n; i++) g[i] = (1.0 - vt) * f[i] + vt * h[i];  /* line 5 */
        for (int64_t i = 0; i < n; i++) r[i] = y[i] - g[i];               /* line 6: L2 pseudo residuals at g */
        int32_t ks, kc;
        double sse, sse_c, gap, gap_c;
        find_best_ws(p, r, w, &ks, theta, &sse, NULL, &gap);              /* line 7 */
        learner_values(p, ks, theta, bcur);
        for (int64_t i = 0; i < n; i++) f[i] = g[i] + J->nu * bcur[i];    /* line 8 */
        if (m > 1) {                                                       /* lines 9-13 */
            double a = (double)m / (double)(m + 1);
            for (int64_t i = 0; i < n; i++) c[i] = r[i] + a * (c[i] - bprev[i]);
        } else {
            for (int64_t i = 0; i < n; i++) c[i] = r[i];
        }
        find_best_ws(p, c, w, &kc, theta_cor, &sse_c, NULL, &gap_c);      /* line 14 */
        double eta = J->gamma * J->nu / vt;                               /* line 15 */
        learner_values(p, kc, theta_cor, bprev);                          /* b_kcor^[m], reused at m+1 */
        for (int64_t i = 0; i < n; i++) h[i] = h[i] + eta * bprev[i];     /* line 16 */
        /* parameter bookkeeping */
        for (int a = 0; a < K * d; a++) tf[a] = (1.0 - vt) * tf[a] + vt * th[a];
        for (int j = 0; j < d; j++) tf[ks * d + j] += J->nu * theta[j];
        for (int j = 0; j < d; j++) th[kc * d + j] += eta * theta_cor[j];
        double rs = 0.0;
        for (int64_t i = 0; i < n; i++) {
            double e = y[i] - f[i];
            rs += 0.5 * e * e;
        }
        size_t t = (size_t)(m - 1) * B + b;
        J->k_trace[t] = ks;
        J->kcor_trace[t] = kc;
        J->sse_trace[t] = sse;
        if (J->sse_cor_trace) J->sse_cor_trace[t] = sse_c;
        J->risk_trace[t] = rs / (double)n;
        if (J->gap_trace) J->gap_trace[t] = gap;
        if (J->gap_cor_trace) J->gap_cor_trace[t] = gap_c;
    }
    if (J->f_out)
        for (int64_t i = 0; i < n; i++) J->f_out[(size_t)b * n + i] = f[i];
    if (J->h_out)
        for (int64_t i = 0; i < n; i++) J->h_out[(size_t)b * n + i] = h[i];
}

static void* acwb_worker(void* arg) {
    acwb_job* J = (acwb_job*)arg;
    int64_t n = J->p->n;
    int d = J->p->d;
    scratch w;
    scratch_init(&w, d, J->p->n_star);
    double* buf = (double*)malloc(sizeof(double) * 7 * n);
    double* theta = (double*)malloc(sizeof(double) * 2 * d);
    for (int b = J->tid; b < J->B; b += J->nth)
        acwb_one(J, b, &w, buf, buf + n, buf + 2 * n, buf + 3 * n, buf + 4 * n, buf + 5 * n, buf + 6 * n, theta,
                 theta + d);
    free(buf);
    free(theta);
    scratch_free(&w);
    return NULL;
}

int orc_train_acwb(const orc_pool* p, const double* Y, int B, double nu, double gamma, int M, int n_threads,
                   double* offset, double* theta_f, double* theta_h, int32_t* k_trace, int32_t* kcor_trace,
                   double* sse_trace, double* sse_cor_trace, double* risk_trace, double* gap_trace,
                   double* gap_cor_trace, double* f_out, double* h_out) {
    if (!p || p->K < 1) return ORC_EEMPTY;
    if (B < 1 || M < 0 || !(nu >= 0.0) || !(gamma >= 0.0)) return ORC_EINVAL;
    for (int64_t a = 0; a < (int64_t)B * p->n; a++)
        if (!isfinite(Y[a])) return ORC_ENONFINITE;
    if (n_threads < 1) n_threads = 1;
    if (n_threads > B) n_threads = B;
    acwb_job* jobs = (acwb_job*)malloc(sizeof(acwb_job) * n_threads);
    pthread_t* thr = (pthread_t*)malloc(sizeof(pthread_t) * n_threads);
    for (int t = 0; t < n_threads; t++) {
        acwb_job J = {p, Y, B, M, t, n_threads, nu, gamma, offset, theta_f, theta_h, sse_trace, sse_cor_trace,
                      risk_trace, gap_trace, gap_cor_trace, f_out, h_out, k_trace, kcor_trace};
        jobs[t] = J;
    }
    for (int t = 1; t < n_threads; t++) pthread_create(&thr[t], NULL, acwb_worker, &jobs[t]);
    acwb_worker(&jobs[0]);
    for (int t = 1; t < n_threads; t++) pthread_join(thr[t], NULL);
    free(jobs);
    free(thr);
    return ORC_OK;
}

/* ------------------------------------------------------------------ HCWB */

/* weighted fit of learner k (w = 0/1 row mask, P:L870 observation weights):
 * theta = (Z^T W Z + lambda D)^-1 Z^T W r, SSE = sum_i w_i (r_i - Z(i) theta)^2 */
static double fit_one_w(const orc_pool* p, int k, const double* r, const double* w, const double* Lw, scratch* ws,
                        double* theta) {
    int d = p->d, n_star = p->n_star;
    int64_t n = p->n;
    const int32_t* idx = p->idx + (size_t)k * n;
    const double* Zb = p->Zb + (size_t)k * n_star * d;
    if (p->mode == ORC_MODE_BINNED) {
        orc_bin_mat_vec(Zb, n_star, d, idx, w, r, n, ws->s);   /* P:L898-904 with weights */
    } else {
        const double* rows = (p->mode == ORC_MODE_DENSE) ? Zb : p->Zx + (size_t)k * n * d;
        dense_ztwr_rows(rows, (p->mode == ORC_MODE_DENSE) ? idx : NULL, d, w, r, n, ws->s);
    }
    chol_fb(Lw + (size_t)k * d * d, d, ws->s, theta);
    double sse = 0.0;
    for (int64_t i = 0; i < n; i++) {
        if (w[i] == 0.0) continue;
        const double* zi = (p->mode == ORC_MODE_UNBINNED) ? p->Zx + ((size_t)k * n + i) * d : Zb + (size_t)idx[i] * d;
        double v = 0.0;
        for (int j = 0; j < d; j++) v += zi[j] * theta[j];
        double e = r[i] - v;
        sse += e * e;
    }
    return sse;
}

static void find_best_w(const orc_pool* p, const double* r, const double* w, const double* Lw, scratch* ws,
                        int32_t* k_out, double* theta_out, double* sse_out, double* gap_out) {
    int d = p->d, best = -1;
    double best_sse = 0.0, second = INFINITY;
    for (int k = 0; k < p->K; k++) {
        double sse = fit_one_w(p, k, r, w, Lw, ws, ws->theta);
        if (best < 0 || sse < best_sse) {
            if (best >= 0) second = best_sse;
            best = k;
            best_sse = sse;
            for (int j = 0; j < d; j++) theta_out[j] = ws->theta[j];
        } else if (sse < second) {
            second = sse;
        }
    }
    *k_out = best;
    *sse_out = best_sse;
    if (gap_out) *gap_out = second - best_sse;
}

typedef struct {
    const orc_pool* p;
    const double* Y;
    const double* wtr;   /* n: 1 = training row, 0 = validation row */
    const double* Ltr;   /* K x d x d: Cholesky of Z^T W Z + lambda D (training rows) */
    int B, M, pat0, tid, nth;
    double nu, gamma;
    double *offset, *theta_f, *sse_trace, *risk_trace, *val_risk_trace, *gap_trace, *gap_cor_trace, *f_out;
    int32_t *k_trace, *kcor_trace, *switch_iter;
} hcwb_job;

/* Algorithm 3 (HCWB): updateACWB (Alg. 2 lines 4-16) on D_train while the
 * validation-risk patience counter is below pat0, then updateCWB (Alg. 1 lines 4-10) on D.
 * Readings: "if pat0 < pat" is read as "while the counter < pat0"; the
 * counter increments when R_emp(f^[m] | D_val) > R_emp(f^[m-1] | D_val), else resets; one
 * pool on D (bins, basis, lambda) with the training fits weighted by the training mask;
 * f^[0] = mean of the training targets; after the switch CWB continues from f. */
static void hcwb_one(const hcwb_job* J, int b, scratch* w, double* f, double* h, double* g, double* r, double* c,
                     double* bprev, double* bcur, double* theta, double* theta_cor, double* th) {
    const orc_pool* p = J->p;
    int64_t n = p->n;
    int d = p->d, K = p->K, B = J->B;
    const double* y = J->Y + (size_t)b * n;
    const double* wt = J->wtr;
    double sy = 0.0, ntr = 0.0, nval = 0.0;
    for (int64_t i = 0; i < n; i++) { sy += wt[i] * y[i]; ntr += wt[i]; nval += 1.0 - wt[i]; }
    double f0 = sy / ntr;
    J->offset[b] = f0;
    for (int64_t i = 0; i < n; i++) { f[i] = f0; h[i] = f0; g[i] = f0; }
    double* tf = J->theta_f + (size_t)b * K * d;
    for (int a = 0; a < K * d; a++) { tf[a] = 0.0; th[a] = 0.0; }
    double vrisk_prev = 0.0;
    for (int64_t i = 0; i < n; i++)
        if (wt[i] == 0.0) { double e = y[i] - f[i]; vrisk_prev += 0.5 * e * e; }
    vrisk_prev /= nval;
    int pat = 0, accel = 1, ma = 0;  /* ma: ACWB iteration counter */
    J->switch_iter[b] = J->M;
    for (int m = 0; m < J->M; m++) {
        int32_t ks, kc = -1;
        double sse, gap, gap_c = 0.0;
        size_t t = (size_t)m * B + b;
        if (accel) {
            ma++;
            double vt = 2.0 / (double)(ma + 1);
            for (int64_t i = 0; i < n; i++) g[i] = (1.0 - vt) * f[i] + vt * h[i];
            for (int64_t i = 0; i < n; i++) r[i] = y[i] - g[i];
            find_best_w(p, r, wt, J->Ltr, w, &ks, theta, &sse, &gap);
            learner_values(p, ks, theta, bcur);
            for (int64_t i = 0; i < n; i++) f[i] = g[i] + J->nu * bcur[i];
            if (ma > 1) {
                double a = (double)ma / (double)(ma + 1);
                for (int64_t i = 0; i < n; i++) c[i] = r[i] + a * (c[i] - bprev[i]);
            } else {
                for (int64_t i = 0; i < n; i++) c[i] = r[i];
            }
            double sse_c;
            find_best_w(p, c, wt, J->Ltr, w, &kc, theta_cor, &sse_c, &gap_c);
            double eta = J->gamma * J->nu / vt;
            learner_values(p, kc, theta_cor, bprev);
            for (int64_t i = 0; i < n; i++) h[i] = h[i] + eta * bprev[i];
            for (int a = 0; a < K * d; a++) tf[a] = (1.0 - vt) * tf[a] + vt * th[a];
            for (int j = 0; j < d; j++) tf[ks * d + j] += J->nu * theta[j];
            for (int j = 0; j < d; j++) th[kc * d + j] += eta * theta_cor[j];
        } else {
            for (int64_t i = 0; i < n; i++) r[i] = y[i] - f[i];
            find_best_ws(p, r, w, &ks, theta, &sse, NULL, &gap);
            learner_values(p, ks, theta, bcur);
            for (int64_t i = 0; i < n; i++) f[i] = f[i] + J->nu * bcur[i];
            for (int j = 0; j < d; j++) tf[ks * d + j] += J->nu * theta[j];
        }
        double rs = 0.0, vr = 0.0;
        for (int64_t i = 0; i < n; i++) {
            double e = y[i] - f[i];
            rs += 0.5 * e * e;
            if (wt[i] == 0.0) vr += 0.5 * e * e;
        }
        vr /= nval;
        if (accel) {  /* Alg. 3 line 6 */
            if (vr > vrisk_prev) pat++;
            else pat = 0;
            if (pat >= J->pat0) { accel = 0; J->switch_iter[b] = m + 1; }
        }
        vrisk_prev = vr;
        J->k_trace[t] = ks;
        J->kcor_trace[t] = kc;
        J->sse_trace[t] = sse;
        J->risk_trace[t] = rs / (double)n;
        J->val_risk_trace[t] = vr;
        if (J->gap_trace) J->gap_trace[t] = gap;
        if (J->gap_cor_trace) J->gap_cor_trace[t] = gap_c;
    }
    if (J->f_out)
        for (int64_t i = 0; i < n; i++) J->f_out[(size_t)b * n + i] = f[i];
}

static void* hcwb_worker(void* arg) {
    hcwb_job* J = (hcwb_job*)arg;
    int64_t n = J->p->n;
    int d = J->p->d, K = J->p->K;
    scratch w;
    scratch_init(&w, d, J->p->n_star);
    double* buf = (double*)malloc(sizeof(double) * 7 * n);
    double* theta = (double*)malloc(sizeof(double) * (2 * d + (size_t)K * d));
    for (int b = J->tid; b < J->B; b += J->nth)
        hcwb_one(J, b, &w, buf, buf + n, buf + 2 * n, buf + 3 * n, buf + 4 * n, buf + 5 * n, buf + 6 * n, theta,
                 theta + d, theta + 2 * d);
    free(buf);
    free(theta);
    scratch_free(&w);
    return NULL;
}

int orc_train_hcwb(const orc_pool* p, const double* Y, int B, const uint8_t* val_mask, double nu, double gamma,
                   int pat0, int M, int n_threads, double* offset, double* theta_f, int32_t* k_trace,
                   int32_t* kcor_trace, double* sse_trace, double* risk_trace, double* val_risk_trace,
                   int32_t* switch_iter, double* gap_trace, double* gap_cor_trace, double* f_out) {
    if (!p || p->K < 1) return ORC_EEMPTY;
    if (B < 1 || M < 0 || pat0 < 1 || !(nu >= 0.0) || !(gamma >= 0.0)) return ORC_EINVAL;
    int64_t n = p->n, ntr = 0;
    int d = p->d, K = p->K;
    for (int64_t a = 0; a < (int64_t)B * n; a++)
        if (!isfinite(Y[a])) return ORC_ENONFINITE;
    double* wtr = (double*)malloc(sizeof(double) * n);
    for (int64_t i = 0; i < n; i++) { wtr[i] = val_mask[i] ? 0.0 : 1.0; ntr += val_mask[i] ? 0 : 1; }
    if (ntr == 0 || ntr == n) { free(wtr); return ORC_EINVAL; }
    /* training-row penalised normal matrices Z^T W Z + lambda D (binMatMat with weights) */
    double* Ltr = (double*)malloc(sizeof(double) * (size_t)K * d * d);
    double* A = (double*)malloc(sizeof(double) * d * d);
    int st = ORC_OK;
    for (int k = 0; k < K && st == ORC_OK; k++) {
        const double* Zb = p->Zb + (size_t)k * p->n_star * d;
        const int32_t* idx = p->idx + (size_t)k * n;
        if (p->mode == ORC_MODE_BINNED) orc_bin_mat_mat(Zb, p->n_star, d, idx, wtr, n, A);
        else {
            const double* rows = (p->mode == ORC_MODE_DENSE) ? Zb : p->Zx + (size_t)k * n * d;
            orc_dense_ztwz(rows, d, (p->mode == ORC_MODE_DENSE) ? idx : NULL, wtr, n, A);
        }
        for (int a = 0; a < d * d; a++) A[a] += p->lambda[k] * p->D[a];
        st = orc_cholesky(A, d, Ltr + (size_t)k * d * d);
    }
    free(A);
    if (st != ORC_OK) { free(wtr); free(Ltr); return ORC_ECALIB; }
    if (n_threads < 1) n_threads = 1;
    if (n_threads > B) n_threads = B;
    hcwb_job* jobs = (hcwb_job*)malloc(sizeof(hcwb_job) * n_threads);
    pthread_t* thr = (pthread_t*)malloc(sizeof(pthread_t) * n_threads);
    for (int t = 0; t < n_threads; t++) {
        hcwb_job J = {p, Y, wtr, Ltr, B, M, pat0, t, n_threads, nu, gamma, offset, theta_f, sse_trace, risk_trace,
                      val_risk_trace, gap_trace, gap_cor_trace, f_out, k_trace, kcor_trace, switch_iter};
        jobs[t] = J;
    }
    for (int t = 1; t < n_threads; t++) pthread_create(&thr[t], NULL, hcwb_worker, &jobs[t]);
    hcwb_worker(&jobs[0]);
    for (int t = 1; t < n_threads; t++) pthread_join(thr[t], NULL);
    free(jobs);
    free(thr);
    free(wtr);
    free(Ltr);
    return ORC_OK;
}

/* -------------------------------------------------------------- predict */

/* ------------------------------------------------------ CV folds (NEXT-4) */

/* Alg. 1 supp. with 0/1 observation weights per replication (binMatMat /
 * binMatVec with weights; the weights of P:L870): replication b fits on the rows
 * whose fold differs from fold_of_rep[b] (all rows when fold_of_rep[b] < 0) and the held-out
 * rows only follow the model.  Per replication, step by step:
 *   f0 = mean of y over its training rows (line 2 on D_train);
 *   r = y - f on every row (line 4), fitted with weights w (w_i = 1 on training rows):
 *   theta_k = (Z_k^T W Z_k + lambda_k D)^-1 Z_k^T W r (lambda of the pool, calibrated on all rows),
 *   SSE_k = sum_i w_i (r_i - (Z_k theta_k)_i)^2 (lines 5-8), k* = argmin (lowest k, line 9);
 *   f += nu Z_k* theta* on every row (line 10), theta_agg[k*] += nu theta* (P:L838);
 *   risk_trace = sum_i w_i (y_i - f_i)^2 / (2 sum w), val_risk_trace = the same over the
 *   held-out rows (0 when there are none). */
typedef struct {
    const orc_pool* p;
    const double* Y;
    const int32_t* fold_of_rep;
    const double* W;    /* F x n weights (fold f held out) */
    const double* Lf;   /* F x K x d x d Cholesky factors of Z^T W_f Z + lambda D */
    int B, M, F, tid, nth;
    double nu;
    double *offset, *theta_agg, *sse_trace, *risk_trace, *val_risk_trace, *gap_trace, *f_out;
    int32_t* k_trace;
} folds_job;

static void folds_one(const folds_job* J, int b, scratch* ws, double* f, double* r, double* theta, const double* ones,
                      const double* Lall) {
    const orc_pool* p = J->p;
    int64_t n = p->n;
    int d = p->d, K = p->K, B = J->B;
    const double* y = J->Y + (size_t)b * n;
    const int fb = J->fold_of_rep[b];
    const double* w = fb < 0 ? ones : J->W + (size_t)fb * n;
    const double* L = fb < 0 ? Lall : J->Lf + (size_t)fb * K * d * d;
    double sw = 0.0, sy = 0.0, sv = 0.0;
    for (int64_t i = 0; i < n; i++) { sw += w[i]; sy += w[i] * y[i]; }
    const double f0 = sy / sw;
    J->offset[b] = f0;
    for (int64_t i = 0; i < n; i++) f[i] = f0;
    double* agg = J->theta_agg + (size_t)b * K * d;
    for (int a = 0; a < K * d; a++) agg[a] = 0.0;
    for (int m = 0; m < J->M; m++) {
        for (int64_t i = 0; i < n; i++) r[i] = y[i] - f[i];
        int32_t ks;
        double sse, gap;
        find_best_w(p, r, w, L, ws, &ks, theta, &sse, &gap);
        const double* Zb = p->Zb + (size_t)ks * p->n_star * d;
        const int32_t* idx = p->idx + (size_t)ks * n;
        for (int64_t i = 0; i < n; i++) {
            const double* zi = (p->mode == ORC_MODE_UNBINNED) ? p->Zx + ((size_t)ks * n + i) * d : Zb + (size_t)idx[i] * d;
            double v = 0.0;
            for (int j = 0; j < d; j++) v += zi[j] * theta[j];
            f[i] = f[i] + J->nu * v;
        }
        for (int j = 0; j < d; j++) agg[ks * d + j] += J->nu * theta[j];
        double rs = 0.0, rv = 0.0;
        sv = 0.0;
        for (int64_t i = 0; i < n; i++) {
            double e = y[i] - f[i];
            rs += w[i] * 0.5 * e * e;
            rv += (1.0 - w[i]) * 0.5 * e * e;
            sv += 1.0 - w[i];
        }
        J->k_trace[(size_t)m * B + b] = ks;
        J->sse_trace[(size_t)m * B + b] = sse;
        J->risk_trace[(size_t)m * B + b] = rs / sw;
        J->val_risk_trace[(size_t)m * B + b] = sv > 0.0 ? rv / sv : 0.0;
        if (J->gap_trace) J->gap_trace[(size_t)m * B + b] = gap;
    }
    if (J->f_out)
        for (int64_t i = 0; i < n; i++) J->f_out[(size_t)b * n + i] = f[i];
}

typedef struct {
    const folds_job* J;
    const double* ones;
    const double* Lall;
} folds_ctx;

static void* folds_worker(void* arg) {
    const folds_ctx* X = (const folds_ctx*)arg;
    const folds_job* J = X->J;
    scratch w;
    scratch_init(&w, J->p->d, J->p->n_star);
    double* f = (double*)malloc(sizeof(double) * J->p->n);
    double* r = (double*)malloc(sizeof(double) * J->p->n);
    double* theta = (double*)malloc(sizeof(double) * J->p->d);
    for (int b = J->tid; b < J->B; b += J->nth) folds_one(J, b, &w, f, r, theta, X->ones, X->Lall);
    free(f); free(r); free(theta);
    scratch_free(&w);
    return NULL;
}

/* penalised normal matrix of learner k with weights w: Z^T W Z + lambda_k D, Cholesky into L */
static int weighted_factor(const orc_pool* p, int k, const double* w, double* A, double* L) {
    int d = p->d;
    int64_t n = p->n;
    const double* Zb = p->Zb + (size_t)k * p->n_star * d;
    const int32_t* idx = p->idx + (size_t)k * n;
    if (p->mode == ORC_MODE_BINNED) orc_bin_mat_mat(Zb, p->n_star, d, idx, w, n, A);
    else {
        const double* rows = (p->mode == ORC_MODE_DENSE) ? Zb : p->Zx + (size_t)k * n * d;
        orc_dense_ztwz(rows, d, (p->mode == ORC_MODE_DENSE) ? idx : NULL, w, n, A);
    }
    for (int a = 0; a < d * d; a++) A[a] += p->lambda[k] * p->D[a];
    return orc_cholesky(A, d, L);
}

int orc_train_folds(const orc_pool* p, const double* Y, int B, const uint8_t* fold_of_row, int F,
                    const int32_t* fold_of_rep, double nu, int M, int n_threads, double* offset, double* theta_agg,
                    int32_t* k_trace, double* sse_trace, double* risk_trace, double* val_risk_trace,
                    double* gap_trace, double* f_out) {
    if (!p || p->K < 1) return ORC_EEMPTY;
    if (B < 1 || M < 0 || !(nu >= 0.0) || F < 1 || F > 255 || !fold_of_row || !fold_of_rep) return ORC_EINVAL;
    int64_t n = p->n;
    int d = p->d, K = p->K;
    for (int64_t a = 0; a < (int64_t)B * n; a++)
        if (!isfinite(Y[a])) return ORC_ENONFINITE;
    for (int b = 0; b < B; b++)
        if (fold_of_rep[b] >= F || fold_of_rep[b] < -1) return ORC_EINVAL;
    for (int64_t i = 0; i < n; i++)
        if (fold_of_row[i] >= F) return ORC_EINVAL;
    double* W = (double*)malloc(sizeof(double) * (size_t)F * n);
    double* ones = (double*)malloc(sizeof(double) * n);
    double* Lf = (double*)malloc(sizeof(double) * (size_t)F * K * d * d);
    double* Lall = (double*)malloc(sizeof(double) * (size_t)K * d * d);
    double* A = (double*)malloc(sizeof(double) * d * d);
    int st = ORC_OK;
    for (int64_t i = 0; i < n; i++) ones[i] = 1.0;
    for (int f = 0; f < F && st == ORC_OK; f++) {
        double cnt = 0.0;
        for (int64_t i = 0; i < n; i++) {
            W[(size_t)f * n + i] = fold_of_row[i] == f ? 0.0 : 1.0;
            cnt += W[(size_t)f * n + i];
        }
        if (cnt == 0.0) st = ORC_EINVAL;  /* a fold holding out every row */
        for (int k = 0; k < K && st == ORC_OK; k++)
            if (weighted_factor(p, k, W + (size_t)f * n, A, Lf + ((size_t)f * K + k) * d * d) != ORC_OK) st = ORC_ECALIB;
    }
    for (int k = 0; k < K && st == ORC_OK; k++)
        if (weighted_factor(p, k, ones, A, Lall + (size_t)k * d * d) != ORC_OK) st = ORC_ECALIB;
    free(A);
    if (st == ORC_OK) {
        if (n_threads < 1) n_threads = 1;
        if (n_threads > B) n_threads = B;
        folds_job* jobs = (folds_job*)malloc(sizeof(folds_job) * n_threads);
        folds_ctx* ctxs = (folds_ctx*)malloc(sizeof(folds_ctx) * n_threads);
        pthread_t* thr = (pthread_t*)malloc(sizeof(pthread_t) * n_threads);
        for (int t = 0; t < n_threads; t++) {
            folds_job J = {p, Y, fold_of_rep, W, Lf, B, M, F, t, n_threads, nu, offset, theta_agg, sse_trace,
                           risk_trace, val_risk_trace, gap_trace, f_out, k_trace};
            jobs[t] = J;
            folds_ctx X = {&jobs[t], ones, Lall};
            ctxs[t] = X;
        }
        for (int t = 1; t < n_threads; t++) pthread_create(&thr[t], NULL, folds_worker, &ctxs[t]);
        folds_worker(&ctxs[0]);
        for (int t = 1; t < n_threads; t++) pthread_join(thr[t], NULL);
        free(jobs); free(ctxs); free(thr);
    }
    free(W); free(ones); free(Lf); free(Lall);
    return st;
}

int orc_predict(const orc_pool* p, const double* Xnew, int64_t m, const double* offset,
                const double* theta_agg, int B, double* out) {
    int d = p->d, K = p->K, n_star = p->n_star;
    if (p->mode == ORC_MODE_UNBINNED) {
        /* unbinned learners: the basis at x itself, x clamped to the training range
         * [min, max] of the learner (reading U2: the binned pool's end-bin rule) */
        double* zr = (double*)malloc(sizeof(double) * d);
        for (int64_t i = 0; i < m; i++)
            for (int k = 0; k < K; k++)
                if (!isfinite(Xnew[(size_t)k * m + i])) { free(zr); return ORC_ENONFINITE; }
        for (int bb = 0; bb < B; bb++)
            for (int64_t i = 0; i < m; i++) {
                double v = offset[bb];
                for (int k = 0; k < K; k++) {
                    double x = Xnew[(size_t)k * m + i];
                    if (x < p->lo[k]) x = p->lo[k];
                    if (x > p->hi[k]) x = p->hi[k];
                    orc_bspline_basis(&x, 1, p->lo[k], p->hi[k], p->degree, p->n_knots, zr);
                    const double* th = theta_agg + ((size_t)bb * K + k) * d;
                    for (int j = 0; j < d; j++) v += zr[j] * th[j];
                }
                out[(size_t)bb * m + i] = v;
            }
        free(zr);
        return ORC_OK;
    }
    int32_t* lix = (int32_t*)malloc(sizeof(int32_t) * (size_t)K * (m > 0 ? m : 1));
    for (int k = 0; k < K; k++) {
        const double* bnd = p->bnd + (size_t)k * (n_star - 1);
        for (int64_t i = 0; i < m; i++) {
            double x = Xnew[(size_t)k * m + i];
            if (!isfinite(x)) { free(lix); return ORC_ENONFINITE; }
            int a = 0, b = n_star - 1;
            while (a < b) {
                int mid = a + (b - a) / 2;
                if (x <= bnd[mid]) b = mid;
                else a = mid + 1;
            }
            lix[(size_t)k * m + i] = a;
        }
    }
    for (int bb = 0; bb < B; bb++)
        for (int64_t i = 0; i < m; i++) {
            double v = offset[bb];
            for (int k = 0; k < K; k++) {
                const double* zr = p->Zb + ((size_t)k * n_star + lix[(size_t)k * m + i]) * d;
                const double* th = theta_agg + ((size_t)bb * K + k) * d;
                for (int j = 0; j < d; j++) v += zr[j] * th[j];
            }
            out[(size_t)bb * m + i] = v;
        }
    free(lix);
    return ORC_OK;
}
