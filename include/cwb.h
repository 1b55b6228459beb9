/*
 * cwb.h -- C ABI of the B200-native binned componentwise-boosting engine
 * (arXiv 2110.03513, "Accelerated Componentwise Gradient Boosting using
 * Efficient Data Representation and Momentum-based Optimization").
 *
 * Citations "P:L<n>" are lines of the paper text PAPER.md (body L751-1217,
 * supplement L246-751).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 * - Every array argument is a DEVICE pointer allocated by the caller (for
 *   instance by torch), except where "host" is written.  The caller owns
 *   inputs and outputs and must keep them alive until the work enqueued on
 *   `stream` has completed.
 * - All arithmetic is IEEE fp64.  Indices are 0-based.
 * - Calls are asynchronous with respect to the host unless stated: they
 *   validate arguments on the host, enqueue kernels on `stream` and return.
 *   Errors found on the device (a constant feature, a non-finite value, an
 *   unreachable df target) are recorded in the context and reported by the
 *   next call that synchronises (cwb_status, cwb_get_lambda, cwb_get_pool).
 * - Every function returns a cwb_code (0 = success); no C++ exception
 *   crosses the ABI.  cwb_last_error() returns the last message.
 * - A cwb_ctx is not thread-safe; use one context per host thread / stream.
 * - Learner k is the univariate binned P-spline base learner of feature k
 *   (K = number of features).
 */
#ifndef CWB_H
#define CWB_H

#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CWB_OK = 0,
    CWB_EINVAL = -1,        /* bad dimension, null pointer, n* < 2, unsupported size        */
    CWB_EDEGENERATE = -2,   /* a feature is constant: min(x) == max(x) (P:L859 undefined)    */
    CWB_ECALIB = -3,        /* df target not reachable (supp. P:L314-319)                     */
    CWB_ENONFINITE = -4,    /* NaN/Inf in x, y or r                                           */
    CWB_EEMPTY = -5,        /* empty base-learner pool (K = 0)                                */
    CWB_ECUDA = -6,         /* CUDA runtime error                                             */
    CWB_ENCCL = -7,         /* communicator error (row-sharded mode)                          */
    CWB_ENOMEM = -8,        /* device allocation failed                                       */
    CWB_EUNSUPPORTED = -9   /* configuration outside what the kernels implement               */
} cwb_code;
/* Error state of a context: a call rejected before any work is enqueued (CWB_EINVAL for
 * its arguments, CWB_EUNSUPPORTED) leaves the context usable; any other error (a device-
 * side status, CUDA, NCCL, allocation) is kept and returned by every later call on it. */

typedef struct cwb_ctx cwb_ctx;

/* Learner configuration ("20 knots and degree 3"; P:L1049 df = 5). */
typedef struct {
    int32_t n_star_rule;  /* 0: n* = ceil(sqrt n), 1: ceil(n^(1/4)), 2: fixed */
    int32_t n_star_fixed; /* n* when n_star_rule == 2 (>= 2)                                      */
    int32_t degree;       /* B-spline degree, 1..3 (default 3)                                    */
    int32_t n_knots;      /* inner knots (default 20); d = n_knots + degree + 1 <= 32             */
    double df;            /* target degrees of freedom per learner (default 5)                   */
    int32_t df_kind;      /* 1: df1 = tr H, 2: df2 = tr(2H - H^2) (supp. P:L314-318)              */
    int32_t batch_hint;   /* expected B of the cwb_train calls (0: unknown).  When > 0, cwb_init
                             builds the fused kernel's gather plan for that B on a side stream,
                             overlapped with the rest of the pool construction.                   */
    int32_t unbinned;     /* 0: binned learners (the paper's method, default).  1: unbinned ("nb")
                             learners on the raw feature values, the
                             baseline binning is compared against: per row 4 non-zero
                             cubic B-spline values at the knot span of x.  Degree 3 only;
                             cwb_train (L2), cwb_find_best and cwb_predict (basis at x clamped
                             to the training range); the other training calls return
                             CWB_EUNSUPPORTED. */
    int32_t train_hint;   /* the training call batch_hint is for, which fixes the shape (threads per
                             CTA, replications per CTA) of the plan cwb_init pre-builds: 0 cwb_train
                             (default), 1 cwb_train_acwb, 2 cwb_train_hcwb, 3 cwb_train_bernoulli.
                             Any call still works on any context; a call whose shape differs from
                             the pre-built plan rebuilds it first.  Out of range: CWB_EINVAL.     */
} cwb_config;

/* Fills *cfg with the paper's defaults: sqrt rule, degree 3, 20 knots, df1 = 5, no batch hint
 * (train_hint 0), binned learners. */
void cwb_default_config(cwb_config* cfg);

/* Library ABI version (major*100 + minor). */
int cwb_version(void);

/* ------------------------------------------------------------------------
 * Stand-alone primitives of Sec. 3.1 (no context).
 * ---------------------------------------------------------------------- */

/* Binning of one feature.
 *   x[n]          feature values.
 *   z_out[n_star] design points z_l = min + l/(n*-1) (max - min), z[n*-1] = max.
 *   bnd_out[n*-1] bin boundaries z_l + (z_{l+1} - z_l)/2 (may be NULL).
 *   idx_out[n]    index vector: smallest l with x <= bnd_l, else n*-1 (a value
 *                 on a boundary goes to the lower bin), stored as uint8
 *                 (idx_bytes = 1, n* <= 256) or uint16 (idx_bytes = 2).
 * Bit-exact with the paper's definition evaluated in fp64 without FMA.
 * Errors: CWB_EINVAL (n < 1, n* < 2, n* too large for idx_bytes),
 * CWB_EDEGENERATE / CWB_ENONFINITE (reported by this call: it synchronises). */
int cwb_bin(const double* x, int64_t n, int32_t n_star, double* z_out, double* bnd_out,
            void* idx_out, int32_t idx_bytes, cudaStream_t stream);

/* Algorithm binMatMat: out (d x d, row-major) = Zb^T diag(c) Zb with
 * c_l = sum_{i: idx(i)=l} w_i (w == NULL: ones).
 *   Zb[n_star][d] reduced design matrix, idx[n] (idx_bytes 1 or 2). */
int cwb_bin_mat_mat(const double* Zb, int32_t n_star, int32_t d, const void* idx, int32_t idx_bytes,
                    const double* w, int64_t n, double* out, cudaStream_t stream);

/* Algorithm binMatVec, for B vectors at once:
 *   R[B][n] (vector b contiguous), out[B][d]: out_b = Zb^T u_b,
 *   u_b(l) = sum_{i: idx(i)=l} w_i R[b][i] (w == NULL: ones).
 * The per-bin sums run in increasing row order (counting-sort inversion of
 * the index vector, computed on the device by this call). */
int cwb_bin_mat_vec(const double* Zb, int32_t n_star, int32_t d, const void* idx, int32_t idx_bytes,
                    const double* w, const double* R, int64_t n, int32_t B, double* out,
                    cudaStream_t stream);

/* ------------------------------------------------------------------------
 * Base-learner pool (init steps I1-I8 of DESIGN.md).
 * ---------------------------------------------------------------------- */

/* Builds the pool of K binned P-spline learners from X[K][n] (feature-major):
 * per learner min/max, the number of bins min(n*, distinct values),
 * design points, index vector, the bin inversion (rows sorted by
 * bin), basis at the design points Zb, G = binMatMat, lambda
 * with df(lambda) = cfg->df (supp. P:L314-319; solved by safeguarded Newton on
 * the definition tr((G + lambda D)^-1 G)) and the cached
 * inverse of G + lambda D.  cfg == NULL uses the defaults.  The
 * context owns all its device buffers (stream-ordered allocations on `stream`).
 * Errors: CWB_EINVAL (n < 2, K < 1, d > 32, degree not in 1..3, n* < 2),
 * CWB_EUNSUPPORTED (n* > 12288 bins per learner: the pool kernels keep per-bin
 * tables in shared memory; cwb_bin alone accepts up to 65536), CWB_EEMPTY
 * (K == 0); device-side errors (constant feature, non-finite x, unreachable
 * df) via cwb_status(). */
int cwb_init(cwb_ctx** ctx, const double* X, int64_t n, int32_t K, const cwb_config* cfg,
             cudaStream_t stream);

/* Synchronises the context's last stream and returns the first recorded
 * error (host or device side), or CWB_OK. */
int cwb_status(cwb_ctx* ctx);

/* Human-readable message of the last error (static storage when ctx == NULL). */
const char* cwb_last_error(const cwb_ctx* ctx);

/* Host outputs: n* and d of the pool, K, n. */
int cwb_get_dims(const cwb_ctx* ctx, int32_t* n_star, int32_t* d, int32_t* K, int64_t* n);

/* Host output lambda[K] (synchronises). */
int cwb_get_lambda(cwb_ctx* ctx, double* lambda_out);

/* Host output n_star_k[K] (synchronises): the bins of every learner, min(n*, number of
 * distinct values of its feature; -0.0 and +0.0 are one value).  S:L143 / SURVEY 8(c)
 * step 1 clamp n* to the distinct values; learner k's design points are those of
 * n*_k bins over [min, max], stored in the first n*_k slots of its z[n*] row
 * (the slots after are padding: z = max, no row binned there).  CWB_EINVAL: NULL
 * output. */
int cwb_get_n_star_k(cwb_ctx* ctx, int32_t* n_star_k_out);

/* Device copies of the pool for inspection (each pointer may be NULL):
 * z[K][n*], idx[K][n] (uint16 regardless of the internal width),
 * Zb[K][n*][d], G[K][d][d], Ainv[K][d][d].  Synchronises. */
int cwb_get_pool(cwb_ctx* ctx, double* z, uint16_t* idx, double* Zb, double* G, double* Ainv);

/* Implementation selector for cwb_train and its variants (tests use it to cover
 * all): 0 = auto (1 when it fits, else 2; never 3), 1 = fused persistent kernel (one
 * CTA per one or two replications, residuals resident in shared memory;
 * CWB_EUNSUPPORTED from the training call when its layout does not fit), 2 = general
 * per-iteration kernels, 3 = cross-Gram formulation (cwb_train only, L2 loss; SURVEY
 * Sec. 7.3 item 3): s_k = Z_k^T r is updated by s_k -= nu (Z_k^T Z_k*) theta* and r^T r
 * by its exact expansion (Alg. 1 supp. line 8, carried through the linear map
 * Z^T), so after one binMatVec pass for the initial residuals an iteration costs
 * O(K d^2) per replication instead of O(n); the cross Gram Z^T Z (K d x K d, built
 * once per pool by binMatVec over the gathered basis rows) is kept in the context.
 * The same iterates as paths 1/2 up to rounding; the residuals themselves are never
 * formed (the outputs do not need them).
 * Errors: CWB_EINVAL (path not 0..3), CWB_EUNSUPPORTED (1 on a row-sharded context; 0 or 1
 * on a learner-sharded context, which runs the per-iteration kernels only; 3 on a sharded or
 * unbinned pool; the training variants other than cwb_train return it for path 3). */
int cwb_set_path(cwb_ctx* ctx, int32_t path);

/* H1 implementation of cwb_find_best for B <= 4 columns (tests and benchmarks
 * compare them): 0 = streaming gather plan (built on the first call, which
 * synchronises the stream; per chunk of 8176 rows the bins of every learner
 * inverted into a gather schedule, binMatVec P:L898-902), falling back to 1
 * when n* > 6144 (the bin sums of a learner group live in 48 KB of shared
 * memory) or on a row-sharded context; 1 = per-warp histograms with
 * __match_any_sync grouping, falling back to the per-iteration kernels where
 * they do not fit.  Errors: CWB_EINVAL (mode not 0 or 1). */
int cwb_set_narrow(cwb_ctx* ctx, int32_t mode);

/* findBestBaselearner (Alg. 1 supp. lines 5-9) for B
 * residual vectors R[B][n]:
 *   k_out[B]        argmin_k SSE_k (lowest k on ties)
 *   theta_out[B][d] fitted parameters of that learner, (G+lambda D)^-1 Zb^T u
 *   sse_out[B]      SSE = sum_i (r_i - Z_k(i) theta)^2 (unpenalised),
 *                   evaluated as r^T r - (2 theta^T s - theta^T G theta).
 * Any output pointer may be NULL. */
int cwb_find_best(cwb_ctx* ctx, const double* R, int32_t B, int32_t* k_out, double* theta_out,
                  double* sse_out, cudaStream_t stream);

/* Vanilla CWB, Alg. 1 supp., L2 loss with L = (y-f)^2/2, for B
 * independent target vectors Y[B][n] sharing X, M iterations, learning rate nu.
 *   offset_out[B]          f0 = mean(y)
 *   theta_agg_out[B][K][d] theta_k = sum_m 1{k = k[m]} nu theta[m]
 *   k_trace[M][B], sse_trace[M][B]  selected learner and its SSE at iteration m
 *   risk_trace[M][B]       empirical risk after the update of iteration m
 * Trace pointers may be NULL.  Returns after enqueueing (no host sync). */
int cwb_train(cwb_ctx* ctx, const double* Y, int32_t B, double nu, int32_t M, double* offset_out,
              double* theta_agg_out, int32_t* k_trace, double* sse_trace, double* risk_trace,
              cudaStream_t stream);

/* Accelerated CWB, Algorithm 2 ("ACWB"), L2 loss, for B target vectors Y[B][n]:
 * primary model f, momentum model h, combined model g = (1 - t_m) f + t_m h with
 * t_m = 2/(m+1); pseudo residuals at g; error-corrected residuals
 * c^[m] = r^[m] + m/(m+1) (c^[m-1] - b_kcor^[m-1]); second findBestBaselearner on c;
 * h += eta_m b_kcor with eta_m = gamma nu / t_m.  Readings: the primary step
 * is nu (the prose's beta), the correction recursion uses the previous correction
 * learner.  Outputs (device):
 *   offset_out[B]
 *   theta_f_out[B][K][d], theta_h_out[B][K][d]  parameters of f and h (bookkeeping of
 *        theta_g = (1-t)theta_f + t theta_h; theta_f = theta_g + nu e_k theta;
 *        theta_h += eta e_kcor theta_cor), so f = offset + sum_k Z_k theta_f[k]
 *   k_trace, kcor_trace [M][B]  learners fitted to r and to c
 *   sse_trace[M][B]             SSE of the fit to r;  risk_trace[M][B]  risk of f
 * Trace pointers may be NULL.  Paper default gamma = 0.0034. */
int cwb_train_acwb(cwb_ctx* ctx, const double* Y, int32_t B, double nu, double gamma, int32_t M,
                   double* offset_out, double* theta_f_out, double* theta_h_out, int32_t* k_trace,
                   int32_t* kcor_trace, double* sse_trace, double* risk_trace, cudaStream_t stream);

/* CWB (Alg. 1 supp.) with the Bernoulli loss of the logistic model,
 * L(y, f) = log(1 + exp(f)) - y f for y in {0, 1} (binary classification, the paper's
 * real-data setting P:L411).  Arguments and outputs as
 * cwb_train, except: offset_out[b] = log(p / (1 - p)) with p = mean(y_b) (Alg. 1 line 2,
 * argmin_c R_emp(c)); the pseudo residuals are r = y - 1 / (1 + exp(-f)), fitted
 * by the base learners with the L2 criterion as for the L2 loss (sse_trace = SSE of that
 * fit); risk_trace[m][b] = mean L(y, f) after the update of iteration m.  The persistent
 * kernel of cwb_train when it fits (y and f in shared memory), else the per-iteration kernels
 * (cwb_set_path selects).  Errors: CWB_EINVAL (arguments; a target value that is not 0
 * or 1, reported by cwb_status), CWB_EDEGENERATE (mean(y_b) is 0 or 1, cwb_status),
 * CWB_ENONFINITE, CWB_EUNSUPPORTED (row-sharded context, unbinned pool). */
int cwb_train_bernoulli(cwb_ctx* ctx, const double* Y, int32_t B, double nu, int32_t M, double* offset_out,
                        double* theta_agg_out, int32_t* k_trace, double* sse_trace, double* risk_trace,
                        cudaStream_t stream);

/* CWB with per-replication cross-validation folds (0/1 observation weights, SURVEY NEXT-4;
 * binMatMat / binMatVec with weights P:L887-904, the weights of P:L870).  fold_of_row[n]
 * (device, uint8, values < F) assigns every row to one of F folds; replication b (fold_of_rep[b],
 * device int32, -1 = no hold-out) fits on the rows of the other folds: offset = mean of its
 * training targets, s = Z^T W r, theta = (Z^T W Z + lambda D)^-1 s with the pool's lambda,
 * SSE over its training rows; the model is updated on every row.  Outputs as cwb_train;
 * risk_trace[m][b] = sum over training rows of (y - f)^2 / (2 n_train), val_risk_trace[m][b] the
 * same over the held-out rows (0 when none).  Per-iteration kernels.  Errors: CWB_EINVAL
 * (arguments; fold ids out of range or a replication without training rows, via cwb_status),
 * CWB_ECALIB (a fold's training rows leave Z^T W Z + lambda D singular), CWB_EUNSUPPORTED
 * (row-sharded context, unbinned pool). */
int cwb_train_folds(cwb_ctx* ctx, const double* Y, int32_t B, const uint8_t* fold_of_row, int32_t F,
                    const int32_t* fold_of_rep, double nu, int32_t M, double* offset_out, double* theta_agg_out,
                    int32_t* k_trace, double* sse_trace, double* risk_trace, double* val_risk_trace,
                    cudaStream_t stream);

/* Hybrid CWB, Algorithm 3 ("HCWB"), L2 loss.  val_mask[n] (device, uint8):
 * 1 = validation row (D_val), 0 = training row (D_train); the split is the caller's
 * (seeded) draw.  Per replication: ACWB (as cwb_train_acwb, momentum gamma) fitted on the
 * training rows while the validation-risk patience counter is below pat0 (the counter
 * increments when R_emp(f^[m] | D_val) > R_emp(f^[m-1] | D_val), resets otherwise;
 * P:L986's "if pat0 < pat" read this way), then CWB on all rows continuing from
 * the primary model f.  One pool (bins, basis, lambda) on all rows; training fits use the
 * training-row G.  Outputs (device): offset_out[B] (mean of the training targets),
 * theta_f_out[B][K][d] (f = offset + sum_k Z_k theta_f[k]); traces [M][B]: k_trace,
 * kcor_trace (-1 after the switch), sse_trace (SSE of the primary fit on its rows),
 * risk_trace (risk of f on all rows), val_risk_trace; switch_iter[B] = first CWB
 * iteration (M if none).  Trace pointers may be NULL.  Paper defaults gamma = 0.037,
 * pat0 = 5.  Errors: CWB_EINVAL (pat0 < 1, val_mask without a training
 * row or without a validation row -- reported by cwb_status, the check runs on the device),
 * CWB_ECALIB. */
int cwb_train_hcwb(cwb_ctx* ctx, const double* Y, int32_t B, const uint8_t* val_mask, double nu, double gamma,
                   int32_t pat0, int32_t M, double* offset_out, double* theta_f_out, int32_t* k_trace,
                   int32_t* kcor_trace, double* sse_trace, double* risk_trace, double* val_risk_trace,
                   int32_t* switch_iter, cudaStream_t stream);

/* Same as cwb_train but every array is a HOST pointer (X[K][n], Y[B][n] in,
 * the rest out); the host<->device copies are enqueued on `stream` and the
 * call synchronises before returning.  Builds and frees its own context. */
int cwb_fit_host(const double* X, int64_t n, int32_t K, const cwb_config* cfg, const double* Y,
                 int32_t B, double nu, int32_t M, double* offset_out, double* theta_agg_out,
                 int32_t* k_trace, double* sse_trace, double* risk_trace, cudaStream_t stream);

/* Prediction with aggregated parameters:
 * out[b][i] = offset[b] + sum_k Zb_k(bin_k(Xnew[k][i]))^T theta_agg[b][k],
 * Xnew[K][m] hashed into the training bins (values outside [min, max] fall
 * into the end bins). */
int cwb_predict(cwb_ctx* ctx, const double* Xnew, int64_t m, const double* offset,
                const double* theta_agg, int32_t B, double* out, cudaStream_t stream);

/* Profiling hook: when cycles4 (a DEVICE buffer of 4 int64) is non-NULL, every
 * later fused cwb_train launch writes the clock64() cycles its CTA 0 spent in
 * the four phases of an iteration (A: binMatVec sums, B: per-learner
 * selection criterion, C: argmax + parameters, D: residual update), summed over
 * the M iterations.  NULL switches it off (default). */
int cwb_set_phase_timing(cwb_ctx* ctx, int64_t* cycles4);

/* Profiling hook of the per-iteration (general) path: with on != 0 every later
 * binMatVec phase H1 (k_h1, or the k_h1c row-chunk launches) is
 * bracketed by a pair of CUDA events recorded on the call's stream (the context
 * owns them).  cwb_get_h1_time synchronises on the last pair, returns the summed
 * elapsed time of every bracketed phase since the last call (*ms_total) and their
 * number (*n_phases, may be NULL), and starts a new tally.  bench.py uses it for the
 * roofline of the dominant kernel of the R3/R4 steps.  Errors: CWB_EINVAL (NULL),
 * CWB_ECUDA. */
int cwb_set_h1_timing(cwb_ctx* ctx, int32_t on);
int cwb_get_h1_time(cwb_ctx* ctx, double* ms_total, int32_t* n_phases);

/* ------------------------------------------------------------- row sharding
 * The rows of the data are partitioned over `world` ranks (one process and GPU
 * each).  binMatVec is linear in the rows -- u(l) is a sum over the rows i of bin l
 * and s = Zb^T u -- and so is r^T r, so each iteration needs
 * the sum over ranks of the per-rank s (K x d per replication) and r^T r: one
 * all-reduce of (K d + 1) x Bp doubles (Bp = B rounded up to 32).  The selection
 * (P:L292), theta, theta_agg and the traces are then the same bytes on every rank,
 * and the residual update touches the local rows only.
 *
 * Every rank calls cwb_init on the FULL X (the pool -- bins, basis, G, lambda,
 * A^-1 -- is a function of all rows; identical on every rank) and then
 * attaches exactly once, before its first cwb_train / cwb_find_best.  From then
 * on the context holds only rows [row_begin, row_end) = [floor(n r / W),
 * floor(n (r + 1) / W)) of the index vectors, cwb_train / cwb_find_best take the
 * LOCAL block Y[B][row_end - row_begin] (R for find_best) and every rank must make
 * the same sequence of calls with the same B, nu and M.  offset = mean over all n
 * rows, risk = r^T r / (2 n) with the global n.  Sums of different rank counts
 * differ in rounding order from the unsharded run (within the parity tolerance).
 * cwb_get_dims then reports the local row count.  cwb_train_acwb / cwb_train_hcwb
 * and the fused path are not available on a row-sharded context
 * (CWB_EUNSUPPORTED).  Errors: CWB_EINVAL (rank outside [0, world), world > n,
 * already attached), CWB_ENCCL (library or communicator failure). */

/* Writes a fresh NCCL unique id (128 bytes, HOST buffer) for cwb_comm_init:
 * call on one rank and send the bytes to the others.  The NCCL library
 * (libnccl.so.2) is loaded on first use; CWB_ENCCL if it cannot be. */
int cwb_comm_unique_id(void* id_out128);

/* A communicator of `world` ranks, this process being `rank`; it may serve any
 * number of contexts (one at a time per stream) and must outlive them.
 * cwb_comm_init: an NCCL communicator, ncclCommInitRank(world, id, rank) on the
 * current device (all ranks call it collectively); the all-reduces are issued
 * on the stream of each cwb_train / cwb_find_best call.
 * cwb_comm_init_fn: the caller's collective.  fn(buf, count, stream, user) must
 * replace the DEVICE array buf[count] (fp64) by its elementwise sum over the
 * world ranks -- the same bytes on every rank -- ordered after the work already
 * on `stream` and before the work enqueued after it returns (it may synchronise
 * the stream), and return 0 (anything else fails the call with CWB_ENCCL).
 * Errors: CWB_EINVAL (rank outside [0, world), NULL arguments), CWB_ENCCL. */
typedef struct cwb_comm cwb_comm;
typedef int (*cwb_allreduce_fn)(double* buf, int64_t count, cudaStream_t stream, void* user);
int cwb_comm_init(cwb_comm** comm, const void* id128, int32_t rank, int32_t world);
int cwb_comm_init_fn(cwb_comm** comm, cwb_allreduce_fn fn, void* user, int32_t rank, int32_t world);

/* Destroys the communicator (NCCL: ncclCommDestroy).  No context attached to it may
 * be used afterwards; work they enqueued must have completed.  comm may be NULL. */
void cwb_comm_free(cwb_comm* comm);

/* Row-shard ctx over comm (borrowed): keeps this rank's row block, as described
 * above.  Once per context, before its first cwb_train / cwb_find_best. */
int cwb_attach_comm(cwb_ctx* ctx, cwb_comm* comm);

/* Learner sharding (the alternative to row sharding): ctx keeps every row and
 * learner (a context built from all of X on every rank), and this rank fits the learners
 * [K rank / world, K (rank+1) / world) in each findBestBaselearner; per iteration one
 * all-reduce (sum) of world x B x (d + 2) doubles gathers every rank's best (delta, k, theta),
 * every rank takes the best over ranks in rank order (the lowest k on ties, as unsharded) and
 * applies the update to its full residuals (replicated, O(n B)).  Results are bitwise those of
 * the unsharded per-iteration kernels.  cwb_train and cwb_find_best only (the other training
 * calls return CWB_EUNSUPPORTED).  Errors: CWB_EINVAL (world > K, already attached). */
int cwb_attach_comm_learners(cwb_ctx* ctx, cwb_comm* comm);

/* Host outputs: first row of this context's block and its row count
 * (0 and n when not sharded), rank and world (0 and 1 when not sharded). */
int cwb_get_rows(const cwb_ctx* ctx, int64_t* row_begin, int64_t* n_rows, int32_t* rank, int32_t* world);

/* Number of kernels this context has launched so far (bench evidence). */
int64_t cwb_launch_count(const cwb_ctx* ctx);

/* Releases every device buffer of the context (stream-ordered on the last
 * stream used).  ctx may be NULL. */
void cwb_free(cwb_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* CWB_H */
