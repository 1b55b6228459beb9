/*
 * cwb_oracle.h -- plain, slow, obviously-correct fp64 CPU oracle for binned
 * componentwise gradient boosting (CWB), arXiv 2110.03513.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2110_03513_b200/) never links, imports or calls it,
 * and it shares no code, header, table or constant generator with the CUDA
 * path.
 *
 * Citations: "P:L<n>" = line n of PAPER.md (the paper body starts at L751,
 * its supplement is L246-751).  Every function below names the passage it
 * follows.  Readings of garbled / silent passages are listed in DESIGN.md
 * ("Readings") and repeated at the function.
 *
 * Conventions: row-major arrays, 0-based indices, int32 bin indices.
 * Learner k uses feature column k (univariate base learners).
 * Return codes mirror include/cwb.h statuses but are defined independently.
 */
#ifndef CWB_ORACLE_H
#define CWB_ORACLE_H
#include <stdint.h>

#define ORC_OK 0
#define ORC_EINVAL (-1)
#define ORC_EDEGENERATE (-2)
#define ORC_ECALIB (-3)
#define ORC_ENONFINITE (-4)
#define ORC_EEMPTY (-5)
#define ORC_ENOMEM (-8)

#define ORC_MODE_DENSE 0    /* materialised rows Z(i)=Zb(idx(i)), fresh Cholesky per fit   */
#define ORC_MODE_BINNED 1   /* Algorithm binMatVec literally, cached Cholesky */
#define ORC_MODE_UNBINNED 2 /* basis evaluated at x itself, no discretisation            */

#ifdef __cplusplus
extern "C" {
#endif

/* n* rule: 0 = ceil(sqrt n) ("n* = sqrt(n)"), 1 = ceil(n^(1/4)),
 * 2 = fixed.  Returns n* or a negative status. */
int orc_n_star(int64_t n, int rule, int fixed);

/* P:L859-861 design points + index vector.  z[n_star], bnd[n_star-1], idx[n]. */
int orc_build_bins(const double* x, int64_t n, int n_star, double* z, double* bnd, int32_t* idx);

/* Basis dimension of a degree-`degree` P-spline with n_knots inner knots. */
int orc_basis_dim(int degree, int n_knots);

/* Cox-de Boor B-spline basis (P-splines of Eilers & Marx) on the
 * extended equidistant knots over [lo, hi].  out is m x d. */
int orc_bspline_basis(const double* x, int64_t m, double lo, double hi, int degree, int n_knots,
                      double* out);

/* Second-order difference penalty D = Delta^T Delta (supp. P:L312). out d x d. */
void orc_penalty(int d, double* D);

/* Algorithm binMatMat: U(idx(i)) += w_i Zb(idx(i)); return U Zb.
 * w == NULL means ones.  out d x d. */
void orc_bin_mat_mat(const double* Zb, int n_star, int d, const int32_t* idx, const double* w,
                     int64_t n, double* out);

/* Algorithm binMatVec: u(idx(i)) += w_i r_i; return Zb^T u.  out d. */
void orc_bin_mat_vec(const double* Zb, int n_star, int d, const int32_t* idx, const double* w,
                     const double* r, int64_t n, double* out);

/* Plain dense products over the materialised discretised design matrix
 * Z(i) = Zb(idx(i)): the definitions binMatMat/binMatVec reach faster. */
void orc_dense_ztwz(const double* Zb, int d, const int32_t* idx, const double* w, int64_t n,
                    double* out);
void orc_dense_ztwr(const double* Zb, int d, const int32_t* idx, const double* w,
                    const double* r, int64_t n, double* out);

/* Plain Cholesky A = L L^T (lower, row-major).  ORC_EINVAL if not SPD. */
int orc_cholesky(const double* A, int d, double* L);
/* Solve A x = b with a fresh Cholesky factorisation. */
int orc_chol_solve(const double* A, int d, const double* b, double* x);

/* Degrees of freedom (supp. P:L314-318) by their definition: df1 = tr(H),
 * df2 = tr(2H - H^2), H = Z (G + lambda D)^-1 Z^T, evaluated with the cyclic
 * trace identity tr(H) = tr((G+lambda D)^-1 G).  kind in {1,2}. */
int orc_df(const double* G, const double* D, int d, double lambda, int kind, double* df_out);

/* Solve df(lambda) = target by bracketing + bisection on the definition
 * (supp. P:L316-319: "must be solved numerically"). */
int orc_df_to_lambda(const double* G, const double* D, int d, double target, int kind,
                     double* lambda_out);

typedef struct {
    int32_t n_star_rule, n_star_fixed, degree, n_knots;
    double df;
    int32_t df_kind;
} orc_config;

/* A pool of K univariate binned P-spline base learners built from X (K x n,
 * feature-major).  Owned by the caller through orc_pool_new / orc_pool_free. */
typedef struct {
    int K, n_star, d, mode;
    int64_t n;
    double* lo;     /* K */
    double* hi;     /* K */
    double* z;      /* K x n_star */
    double* bnd;    /* K x (n_star-1) */
    int32_t* idx;   /* K x n */
    double* Zb;     /* K x n_star x d   (binned / dense modes) */
    double* Zx;     /* K x n x d        (unbinned mode only)   */
    double* G;      /* K x d x d   Z^T Z */
    double* D;      /* d x d */
    double* lambda; /* K */
    double* L;      /* K x d x d   Cholesky of G + lambda D (binned mode cache) */
    int degree, n_knots;  /* of the basis (unbinned prediction evaluates it at new x) */
    int32_t* nsk;   /* K: effective bins of learner k = min(n_star, #distinct x values) (S:L143,
                     * reading N1); design points l >= nsk[k] are padding (z = hi, bnd = +inf,
                     * never hit by a row) */
} orc_pool;

/* Number of distinct values of x (n >= 1), -0.0 and +0.0 counted once: sort a copy, count runs. */
int64_t orc_count_distinct(const double* x, int64_t n);

int orc_pool_new(const double* X, int64_t n, int K, const orc_config* cfg, int mode, orc_pool** out);
void orc_pool_free(orc_pool* p);

/* findBestBaselearner (Alg. 1 supp. lines 5-9) on one
 * residual vector r (n).  Fits every learner, SSE_k = sum_i (r_i - Z_k(i) theta_k)^2
 * (unpenalised), argmin with the lowest k on ties.  gap_out (optional)
 * = SSE of the second best minus SSE of the best. */
int orc_find_best(const orc_pool* p, const double* r, int32_t* k_out, double* theta_out,
                  double* sse_out, double* sse_all_out, double* gap_out);

/* Vanilla CWB, Alg. 1 supp., L2 loss with the 1/2 convention
 * (r = y - f), for B independent target vectors Y (B x n) sharing X.
 * Outputs: offset[B], theta_agg[B][K][d] (theta_k = sum_m 1{k=k[m]} nu theta[m],
 * P:L838 with nu), k_trace/sse_trace/risk_trace/gap_trace[M][B] (risk after
 * the update of iteration m, R_emp = mean 1/2 (y-f)^2), f_out[B][n]
 * (optional final fit).  n_threads >= 1 threads over replications. */
int orc_train(const orc_pool* p, const double* Y, int B, double nu, int M, int n_threads,
              double* offset, double* theta_agg, int32_t* k_trace, double* sse_trace,
              double* risk_trace, double* gap_trace, double* f_out);

/* orc_train (L2) in tie-following mode: at iteration m, replication b takes
 * the learner follow[m][b] instead of its own argmin when that learner's SSE exceeds the minimum
 * by at most tie_rtol * SSE_min (a near-tie: several selections are correct); followed[b] counts
 * those iterations.  Any other difference is kept (the comparator then reports it). */
int orc_train_follow(const orc_pool* p, const double* Y, int B, double nu, int M, int n_threads,
                     const int32_t* follow, double tie_rtol, double* offset, double* theta_agg, int32_t* k_trace,
                     double* sse_trace, double* risk_trace, double* gap_trace, double* f_out, int32_t* followed);

/* orc_train with a loss: ORC_LOSS_L2 (as orc_train) or ORC_LOSS_BERNOULLI, y in {0, 1}:
 * L(y, f) = log(1 + exp(f)) - y f, pseudo residuals r = y - 1/(1 + exp(-f))
 * (P:L833), offset log(p/(1-p)) with p = mean(y) (Alg. 1 line 2),
 * risk_trace = mean L after the update of iteration m.  ORC_EINVAL if some y is not 0
 * or 1, ORC_EDEGENERATE if mean(y) is 0 or 1. */
#define ORC_LOSS_L2 0
#define ORC_LOSS_BERNOULLI 1
int orc_train_loss(const orc_pool* p, const double* Y, int B, int loss, double nu, int M, int n_threads,
                   double* offset, double* theta_agg, int32_t* k_trace, double* sse_trace,
                   double* risk_trace, double* gap_trace, double* f_out);

/* CWB with 0/1 observation weights per replication (cross-validation folds):
 * replication b fits on the rows with fold_of_row[i] != fold_of_rep[b] (every row when
 * fold_of_rep[b] = -1) with G = Z^T W Z and s = Z^T W r (binMatMat / binMatVec with weights,
 * P:L887-904) and the pool's lambda; the held-out rows follow the model.  Outputs as
 * orc_train; offset = mean of y over the training rows; risk_trace / val_risk_trace = half
 * mean squared error over the training / held-out rows after iteration m (0 if none held out).
 * ORC_EINVAL for fold ids >= F, F outside 1..255, a fold holding out every row. */
int orc_train_folds(const orc_pool* p, const double* Y, int B, const uint8_t* fold_of_row, int F,
                    const int32_t* fold_of_rep, double nu, int M, int n_threads, double* offset, double* theta_agg,
                    int32_t* k_trace, double* sse_trace, double* risk_trace, double* val_risk_trace,
                    double* gap_trace, double* f_out);

/* Accelerated CWB, Algorithm 2, L2 loss, for B target vectors: primary
 * model f, momentum model h, combined model g = (1 - theta_m) f + theta_m h, theta_m =
 * 2/(m+1); pseudo residuals at g; error-corrected residuals c; eta_m = gamma nu / theta_m.
 * Outputs: offset[B]; theta_f, theta_h [B][K][d] (parameter bookkeeping of P:L966);
 * traces [M][B]: k (primary learner), kcor (correction learner), SSE of both fits, risk of
 * f after iteration m, SSE gaps to the second best (ties); f_out, h_out [B][n] optional. */
int orc_train_acwb(const orc_pool* p, const double* Y, int B, double nu, double gamma, int M, int n_threads,
                   double* offset, double* theta_f, double* theta_h, int32_t* k_trace, int32_t* kcor_trace,
                   double* sse_trace, double* sse_cor_trace, double* risk_trace, double* gap_trace,
                   double* gap_cor_trace, double* f_out, double* h_out);

/* Hybrid CWB, Algorithm 3: ACWB on the training rows (val_mask[i] == 0) while
 * the validation-risk patience counter is below pat0, then CWB on all rows.  Outputs:
 * offset[B] (mean of the training targets), theta_f[B][K][d] (final primary model);
 * traces [M][B]: k (primary / CWB learner), kcor (-1 after the switch), SSE of the primary fit
 * (training rows before the switch), risk of f on all rows, validation risk of f, SSE gaps;
 * switch_iter[B] = first CWB iteration (0-based; M if none); f_out[B][n] optional. */
int orc_train_hcwb(const orc_pool* p, const double* Y, int B, const uint8_t* val_mask, double nu, double gamma,
                   int pat0, int M, int n_threads, double* offset, double* theta_f, int32_t* k_trace,
                   int32_t* kcor_trace, double* sse_trace, double* risk_trace, double* val_risk_trace,
                   int32_t* switch_iter, double* gap_trace, double* gap_cor_trace, double* f_out);

/* Prediction with the aggregated parameters (P:L822-826 additivity):
 * f(x) = offset + sum_k g_k(z(x))^T theta_k, x hashed into the training bins
 * (clamped to the end bins outside [lo, hi]).  Xnew K x m; out B x m. */
int orc_predict(const orc_pool* p, const double* Xnew, int64_t m, const double* offset,
                const double* theta_agg, int B, double* out);

#ifdef __cplusplus
}
#endif
#endif
