// cwb_abi.cu -- extern "C" entry points declared in include/cwb.h.
// Host-side argument validation, buffer ownership and path selection; every
// arithmetic step of the method runs in the kernels of cwb_init.cu,
// cwb_fused.cu and cwb_iter.cu.  There is no CPU fallback.
#include <cuda_runtime.h>
#include <cstdlib>
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>

#include <mutex>
#include <string>

#include "cwb_internal.cuh"

static thread_local std::string g_err;  // last error of context-free calls

int cwb_bin_mat_vec_impl(const double* Zb, int32_t ns, int32_t d, const void* idx, int32_t idx_bytes,
                         const double* w, const double* R, int64_t n, int32_t B, double* out,
                         cudaStream_t s);
int cwb_bin_mat_mat_impl(const double* Zb, int32_t ns, int32_t d, const void* idx, int32_t idx_bytes,
                         const double* w, int64_t n, double* out, cudaStream_t s);
int cwb_launch_bin_only(cwb_ctx* ctx, int* st, const double* x, int64_t n, int32_t K, int32_t ns,
                        double* lo, double* hi, double* z, double* bnd, void* idx, int32_t idx_bytes,
                        cudaStream_t s, int32_t* nsk = nullptr);

int cwb_num_sms() {
    static int sms = [] {
        int dev = 0, v = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v < 1)
            v = 148;
        return std::min(v, CWB_MAX_SMS);
    }();
    return sms;
}

int cwb_set_error(cwb_ctx* ctx, int code, const std::string& msg) {
    if (ctx) {
        // argument / unsupported-configuration rejections leave the context usable (include/cwb.h)
        if (ctx->status == CWB_OK && code != CWB_EINVAL && code != CWB_EUNSUPPORTED) ctx->status = code;
        ctx->err = msg;
    } else {
        g_err = msg;
    }
    return code;
}

int cwb_check_launch(cwb_ctx* ctx, const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cwb_set_error(ctx, CWB_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return CWB_OK;
}

cudaError_t cwb_alloc(void** p, size_t bytes, cudaStream_t s) {
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;  // keep freed blocks cached in the pool across calls
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    });
    *p = nullptr;
    if (bytes == 0) bytes = 16;
    return cudaMallocAsync(p, bytes, s);
}

void cwb_release(void* p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

void cwb_pool_release(cwb_ctx* c, void* p, cudaStream_t s) {
    const char* a = (const char*)c->arena;
    if (p && !(a && (const char*)p >= a && (const char*)p < a + c->arena_bytes)) cudaFreeAsync(p, s);
}

static const char* status_name(int c) {
    switch (c) {
        case CWB_OK: return "ok";
        case CWB_EINVAL: return "invalid argument";
        case CWB_EDEGENERATE: return "constant feature (min == max)";
        case CWB_ECALIB: return "df target not reachable";
        case CWB_ENONFINITE: return "non-finite input";
        case CWB_EEMPTY: return "empty base-learner pool";
        case CWB_ECUDA: return "CUDA error";
        case CWB_ENCCL: return "communicator error";
        case CWB_ENOMEM: return "out of device memory";
        case CWB_EUNSUPPORTED: return "unsupported configuration";
    }
    return "unknown";
}

// n* rule of P:L859 (sqrt) / P:L445 (fourth root), integer ceiling
static int64_t isqrt_ceil(int64_t n) {
    int64_t s = (int64_t)ceil(sqrt((double)n));
    while (s > 1 && (s - 1) * (s - 1) >= n) s--;
    while (s * s < n) s++;
    return s;
}

static int64_t n_star_of(int64_t n, const cwb_config& c) {
    if (c.n_star_rule == 2) return c.n_star_fixed;
    if (c.n_star_rule == 0) return std::max<int64_t>(2, isqrt_ceil(n));
    if (c.n_star_rule == 1) return std::max<int64_t>(2, isqrt_ceil(isqrt_ceil(n)));
    return -1;
}

extern "C" {

void cwb_default_config(cwb_config* cfg) {
    if (!cfg) return;
    cfg->n_star_rule = 0;
    cfg->n_star_fixed = 0;
    cfg->degree = 3;
    cfg->n_knots = 20;
    cfg->df = 5.0;
    cfg->df_kind = 1;
    cfg->batch_hint = 0;
    cfg->unbinned = 0;
    cfg->train_hint = 0;
}

int cwb_version(void) { return 100; }

const char* cwb_last_error(const cwb_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

int cwb_bin(const double* x, int64_t n, int32_t n_star, double* z_out, double* bnd_out, void* idx_out,
            int32_t idx_bytes, cudaStream_t s) {
    if (!x || !z_out || !idx_out || n < 1 || n_star < 2 || (idx_bytes != 1 && idx_bytes != 2))
        return cwb_set_error(nullptr, CWB_EINVAL, "cwb_bin: invalid argument");
    if ((idx_bytes == 1 && n_star > 256) || n_star > 65536)
        return cwb_set_error(nullptr, CWB_EINVAL, "cwb_bin: n* too large for idx_bytes");
    double *lo = nullptr, *hi = nullptr, *bnd = bnd_out;
    int* st = nullptr;
    bool ok = cwb_alloc((void**)&lo, 8, s) == cudaSuccess && cwb_alloc((void**)&hi, 8, s) == cudaSuccess &&
              cwb_alloc((void**)&st, sizeof(int), s) == cudaSuccess;
    if (ok && !bnd) ok = cwb_alloc((void**)&bnd, sizeof(double) * (n_star - 1), s) == cudaSuccess;
    int rc = ok ? CWB_OK : CWB_ENOMEM;
    if (rc == CWB_OK) {
        cudaMemsetAsync(st, 0, sizeof(int), s);
        rc = cwb_launch_bin_only(nullptr, st, x, n, 1, n_star, lo, hi, z_out, bnd, idx_out, idx_bytes, s);
    }
    int dev_status = 0;
    if (rc == CWB_OK) {
        if (cudaMemcpyAsync(&dev_status, st, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            rc = cwb_set_error(nullptr, CWB_ECUDA, "cwb_bin: synchronisation failed");
    }
    cwb_release(lo, s); cwb_release(hi, s); cwb_release(st, s);
    if (bnd != bnd_out) cwb_release(bnd, s);
    if (rc == CWB_OK && dev_status) rc = cwb_set_error(nullptr, dev_status, std::string("cwb_bin: ") + status_name(dev_status));
    return rc;
}

int cwb_bin_mat_mat(const double* Zb, int32_t n_star, int32_t d, const void* idx, int32_t idx_bytes,
                    const double* w, int64_t n, double* out, cudaStream_t s) {
    if (!Zb || !idx || !out || n < 1 || n > INT32_MAX || n_star < 1 || d < 1 || (idx_bytes != 1 && idx_bytes != 2))
        return cwb_set_error(nullptr, CWB_EINVAL, "cwb_bin_mat_mat: invalid argument");
    int rc = cwb_bin_mat_mat_impl(Zb, n_star, d, idx, idx_bytes, w, n, out, s);
    if (rc) return cwb_set_error(nullptr, rc, std::string("cwb_bin_mat_mat: ") + status_name(rc));
    return CWB_OK;
}

int cwb_bin_mat_vec(const double* Zb, int32_t n_star, int32_t d, const void* idx, int32_t idx_bytes,
                    const double* w, const double* R, int64_t n, int32_t B, double* out, cudaStream_t s) {
    if (!Zb || !idx || !R || !out || n < 1 || n > INT32_MAX || n_star < 1 || d < 1 || B < 1 ||
        (idx_bytes != 1 && idx_bytes != 2))
        return cwb_set_error(nullptr, CWB_EINVAL, "cwb_bin_mat_vec: invalid argument");
    int rc = cwb_bin_mat_vec_impl(Zb, n_star, d, idx, idx_bytes, w, R, n, B, out, s);
    if (rc) return cwb_set_error(nullptr, rc, std::string("cwb_bin_mat_vec: ") + status_name(rc));
    return CWB_OK;
}

void cwb_free(cwb_ctx* c) {
    if (!c) return;
    cudaStream_t s = c->stream;
    if (c->ev_plan) cudaStreamWaitEvent(s, c->ev_plan, 0);  // a plan still building on the side stream
    void* bufs[] = {c->d_status, c->lo, c->hi, c->z, c->bnd, c->idx, c->cnt, c->off, c->perm, c->Zb,
                    c->zj0, c->Zs, c->lwin, c->G, c->Ainv, c->lambda, c->ws.Rt, c->ws.U,
                    c->ws.theta, c->ws.delta, c->ws.rr, c->ws.zhat, c->ws.kstar, c->ws.part, c->ws.narrow, c->ws.colpart, c->ws.acwb, c->ws.pack, c->ws.bern, c->ws.fold, c->ws.lbuf, c->plan, c->permt,
                    c->Cb, c->ZT, c->nsk};
    for (void* p : bufs) cwb_pool_release(c, p, s);
    cwb_release(c->arena, s);
    cwb_stream_release(c, s);
    cwb_nb_release(c, s);
    cwb_release(c->h1c, s);
    cwb_release(c->xg, s);
    if (c->ev_plan) {
        cudaEventSynchronize(c->ev_plan);  // the header copy into the pinned slot has landed
        cudaEventDestroy(c->ev_plan);
    }
    if (c->ev_csr) cudaEventDestroy(c->ev_csr);
    for (cudaEvent_t e : c->h1_ev) cudaEventDestroy(e);
    cwb_release_header_slot(c->h_hdr);
    // c->s2 is the device's shared side stream: not destroyed
    delete c;
}

int cwb_init(cwb_ctx** out, const double* X, int64_t n, int32_t K, const cwb_config* cfg_in,
             cudaStream_t s) {
    if (!out) return cwb_set_error(nullptr, CWB_EINVAL, "cwb_init: ctx pointer is NULL");
    *out = nullptr;
    if (K == 0) return cwb_set_error(nullptr, CWB_EEMPTY, "cwb_init: empty base-learner pool");
    if (!X || n < 2 || K < 0) return cwb_set_error(nullptr, CWB_EINVAL, "cwb_init: invalid argument");
    cwb_config cfg;
    if (cfg_in) cfg = *cfg_in;
    else cwb_default_config(&cfg);
    const int64_t ns = n_star_of(n, cfg);
    const int d = cfg.n_knots + cfg.degree + 1;
    if (ns < 2 || ns > 65536) return cwb_set_error(nullptr, CWB_EINVAL, "cwb_init: n* out of range");
    if (ns > CWB_POOL_MAX_NSTAR)  // per-bin tables of the pool kernels live in shared memory
        return cwb_set_error(nullptr, CWB_EUNSUPPORTED, "cwb_init: n* > 12288 bins per learner");
    if (cfg.degree < 1 || cfg.degree > 3 || cfg.n_knots < 0 || d > CWB_MAX_D)
        return cwb_set_error(nullptr, CWB_EINVAL, "cwb_init: need degree 1..3 and d <= 32");
    if (cfg.df_kind != 1 && cfg.df_kind != 2) return cwb_set_error(nullptr, CWB_EINVAL, "cwb_init: df_kind");
    if (n > INT32_MAX) return cwb_set_error(nullptr, CWB_EUNSUPPORTED, "cwb_init: n >= 2^31");
    if (cfg.unbinned != 0 && cfg.unbinned != 1) return cwb_set_error(nullptr, CWB_EINVAL, "cwb_init: unbinned");
    if (cfg.unbinned && (cfg.degree != 3 || cfg.n_knots + 1 > 255))
        return cwb_set_error(nullptr, CWB_EUNSUPPORTED, "cwb_init: unbinned learners need degree 3");
    if (cfg.train_hint < 0 || cfg.train_hint > 3) return cwb_set_error(nullptr, CWB_EINVAL, "cwb_init: train_hint");
    cwb_ctx* c = new cwb_ctx();
    c->n = n; c->K = K; c->n_star = (int32_t)ns; c->d = d; c->degree = cfg.degree; c->n_knots = cfg.n_knots;
    c->df = cfg.df; c->df_kind = cfg.df_kind;
    c->batch_hint = cfg.batch_hint > 0 && !cfg.unbinned ? cfg.batch_hint : 0;
    c->train_hint = cfg.train_hint;
    c->nb = cfg.unbinned != 0;
    if (const char* e = getenv("CWB_H1_CHUNKING")) c->h1_chunking = atoi(e);  // A/B measurement switch
    if (const char* e = getenv("CWB_H1_WIDE")) c->h1_wide = atoi(e) != 0;       // A/B: k_h1w vs k_h1
    if (c->nb) c->path = 2;  // per-iteration kernels only
    c->idx_bytes = ns <= 256 ? 1 : 2;
    c->perm_bytes = n <= 65536 ? 2 : 4;
    c->stream = s;
    const size_t Ks = K, nn = n, nss = ns, dd = d;
    c->nsp = (int32_t)((ns + 1) / 2 * 2);
    // design points in the support of one B-spline ((degree+1) knot intervals), +2 for rounding
    c->W = (int32_t)std::min<int64_t>(ns, ((int64_t)(cfg.degree + 1) * (ns - 1)) / (cfg.n_knots + 1) + 2);
    // the pool's buffers are carved from one allocation (one host call instead of 18)
    struct Part { void** p; size_t bytes; };
    const Part parts[] = {
        {(void**)&c->d_status, sizeof(int)}, {(void**)&c->lo, 8 * Ks}, {(void**)&c->hi, 8 * Ks},
        {(void**)&c->z, 8 * Ks * nss}, {(void**)&c->bnd, 8 * Ks * (nss - 1)},
        {&c->idx, (size_t)c->idx_bytes * Ks * nn + 16},  // +16: bulk-copy slack
        {(void**)&c->cnt, 4 * Ks * nss}, {(void**)&c->off, 4 * Ks * (nss + 1)},
        {&c->perm, (size_t)c->perm_bytes * (Ks * nn + 8)},  // +8: vector-load padding
        {(void**)&c->Zb, 8 * Ks * nss * dd}, {(void**)&c->zj0, 4 * Ks * nss}, {(void**)&c->Zs, 8 * Ks * nss * CWB_SPW},
        {(void**)&c->lwin, 4 * Ks * dd * 2}, {(void**)&c->G, 8 * Ks * dd * dd}, {(void**)&c->Ainv, 8 * Ks * dd * dd},
        {(void**)&c->lambda, 8 * Ks}, {(void**)&c->Cb, 8 * Ks * dd * 4}, {(void**)&c->ZT, 8 * Ks * (size_t)c->W * dd},
        {(void**)&c->nsk, 4 * Ks}};
    size_t total = 0;
    for (const Part& q : parts) total += (q.bytes + 255) & ~(size_t)255;
    bool ok = cwb_alloc(&c->arena, total, s) == cudaSuccess;
    if (ok) {
        c->arena_bytes = total;
        char* base = (char*)c->arena;
        for (const Part& q : parts) {
            *q.p = base;
            base += (q.bytes + 255) & ~(size_t)255;
        }
    }
    if (!ok) {
        cwb_free(c);
        return cwb_set_error(nullptr, CWB_ENOMEM, "cwb_init: device allocation failed");
    }
    cudaMemsetAsync(c->d_status, 0, sizeof(int), s);
    cudaMemsetAsync(c->perm, 0, (size_t)c->perm_bytes * (Ks * nn + 8), s);
    int rc = cwb_launch_init(c, X, s);
    if (rc) {
        std::string m = c->err;
        cwb_free(c);
        return cwb_set_error(nullptr, rc, m);
    }
    *out = c;
    return CWB_OK;
}

int cwb_status(cwb_ctx* c) {
    if (!c) return cwb_set_error(nullptr, CWB_EINVAL, "cwb_status: NULL context");
    if (c->status) return c->status;
    if (c->ev_plan) cudaEventSynchronize(c->ev_plan);
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return cwb_set_error(c, CWB_ECUDA, cudaGetErrorString(e));
    int dev = 0;
    e = cudaMemcpy(&dev, c->d_status, sizeof(int), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cwb_set_error(c, CWB_ECUDA, cudaGetErrorString(e));
    if (dev) {  // device-side errors are kept whatever their code
        cwb_set_error(c, dev, std::string("device: ") + status_name(dev));
        if (c->status == CWB_OK) c->status = dev;
        return dev;
    }
    return CWB_OK;
}

int cwb_get_dims(const cwb_ctx* c, int32_t* n_star, int32_t* d, int32_t* K, int64_t* n) {
    if (!c) return cwb_set_error(nullptr, CWB_EINVAL, "cwb_get_dims: NULL context");
    if (n_star) *n_star = c->n_star;
    if (d) *d = c->d;
    if (K) *K = c->K;
    if (n) *n = c->n;
    return CWB_OK;
}

int cwb_get_lambda(cwb_ctx* c, double* lambda_out) {
    int rc = cwb_status(c);
    if (rc) return rc;
    if (!lambda_out) return cwb_set_error(c, CWB_EINVAL, "cwb_get_lambda: NULL output");
    CWB_CUDA_TRY(c, cudaMemcpy(lambda_out, c->lambda, sizeof(double) * c->K, cudaMemcpyDeviceToHost));
    return CWB_OK;
}

int cwb_get_n_star_k(cwb_ctx* c, int32_t* out) {
    int rc = cwb_status(c);
    if (rc) return rc;
    if (!out) return cwb_set_error(c, CWB_EINVAL, "cwb_get_n_star_k: NULL output");
    CWB_CUDA_TRY(c, cudaMemcpy(out, c->nsk, sizeof(int32_t) * c->K, cudaMemcpyDeviceToHost));
    return CWB_OK;
}

namespace {
__global__ void k_widen_idx(const uint8_t* a, uint16_t* b, int64_t cnt) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}
}  // namespace

int cwb_get_pool(cwb_ctx* c, double* z, uint16_t* idx, double* Zb, double* G, double* Ainv) {
    int rc = cwb_status(c);
    if (rc) return rc;
    const size_t K = c->K, n = c->n, ns = c->n_star, d = c->d;
    if (z) CWB_CUDA_TRY(c, cudaMemcpy(z, c->z, 8 * K * ns, cudaMemcpyDeviceToDevice));
    if (Zb) CWB_CUDA_TRY(c, cudaMemcpy(Zb, c->Zb, 8 * K * ns * d, cudaMemcpyDeviceToDevice));
    if (G) CWB_CUDA_TRY(c, cudaMemcpy(G, c->G, 8 * K * d * d, cudaMemcpyDeviceToDevice));
    if (Ainv) CWB_CUDA_TRY(c, cudaMemcpy(Ainv, c->Ainv, 8 * K * d * d, cudaMemcpyDeviceToDevice));
    if (idx) {
        if (c->idx_bytes == 2) CWB_CUDA_TRY(c, cudaMemcpy(idx, c->idx, 2 * K * n, cudaMemcpyDeviceToDevice));
        else {
            k_widen_idx<<<1184, 256>>>((const uint8_t*)c->idx, idx, (int64_t)(K * n));
            c->launches++;
            CWB_CUDA_TRY(c, cudaDeviceSynchronize());
        }
    }
    return CWB_OK;
}

int cwb_set_narrow(cwb_ctx* c, int32_t mode) {
    if (!c || mode < 0 || mode > 1) return cwb_set_error(c, CWB_EINVAL, "cwb_set_narrow: invalid argument");
    c->narrow_mode = mode;
    return CWB_OK;
}

int cwb_set_path(cwb_ctx* c, int32_t path) {
    if (!c || path < 0 || path > 3) return cwb_set_error(c, CWB_EINVAL, "cwb_set_path: invalid argument");
    if (c->rows && path == 1) return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_set_path: row-sharded context");
    if (path == 3 && (c->rows || c->lshard || c->nb))
        return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_set_path: the cross-Gram path needs an unsharded binned pool");
    // learner sharding runs on the per-iteration kernels only (the fused and stream paths fit all K learners)
    if (c->lshard && path != 2)
        return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_set_path: learner-sharded context (path 2 only)");
    c->path = path;
    return CWB_OK;
}

int cwb_find_best(cwb_ctx* c, const double* R, int32_t B, int32_t* k_out, double* theta_out,
                  double* sse_out, cudaStream_t s) {
    if (!c || !R || B < 1) return cwb_set_error(c, CWB_EINVAL, "cwb_find_best: invalid argument");
    if (c->status) return c->status;
    c->stream = s;
    if (c->rows) return cwb_find_best_rows(c, R, B, k_out, theta_out, sse_out, s);
    return cwb_find_best_general(c, R, B, k_out, theta_out, sse_out, s);
}

int cwb_train(cwb_ctx* c, const double* Y, int32_t B, double nu, int32_t M, double* offset_out,
              double* theta_agg_out, int32_t* k_trace, double* sse_trace, double* risk_trace,
              cudaStream_t s) {
    if (!c || !Y || !theta_agg_out || B < 1 || M < 0 || !(nu >= 0.0) || !isfinite(nu))
        return cwb_set_error(c, CWB_EINVAL, "cwb_train: invalid argument");
    if (c->status) return c->status;
    c->stream = s;
    if (c->rows)
        return cwb_train_rows(c, Y, B, nu, M, offset_out, theta_agg_out, k_trace, sse_trace, risk_trace, s);
    if (c->path == 3)
        return cwb_train_gram(c, Y, B, nu, M, offset_out, theta_agg_out, k_trace, sse_trace, risk_trace, s);
    if (c->path != 2) {
        bool launched = false;
        int rc = cwb_train_fused(c, Y, B, nu, M, offset_out, theta_agg_out, k_trace, sse_trace,
                                 risk_trace, s, &launched);
        if (rc || launched) return rc;
        if (c->path == 1)
            return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_train: fused path needs more shared memory than a CTA has");
    }
    return cwb_train_general(c, Y, B, nu, M, offset_out, theta_agg_out, k_trace, sse_trace, risk_trace, s);
}

int cwb_train_bernoulli(cwb_ctx* c, const double* Y, int32_t B, double nu, int32_t M, double* offset_out,
                        double* theta_agg_out, int32_t* k_trace, double* sse_trace, double* risk_trace,
                        cudaStream_t s) {
    if (!c || !Y || !theta_agg_out || B < 1 || M < 0 || !(nu >= 0.0) || !isfinite(nu))
        return cwb_set_error(c, CWB_EINVAL, "cwb_train_bernoulli: invalid argument");
    if (c->status) return c->status;
    c->stream = s;
    if (c->rows) return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_train_bernoulli: row-sharded context");
    if (c->lshard) return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_train_bernoulli: learner-sharded context");
    if (c->path == 3) return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_train_bernoulli: the cross-Gram path (3) is cwb_train only");
    if (c->nb) return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_train_bernoulli: unbinned pool (cwb_train only)");
    if (c->path != 2) {
        bool launched = false;
        int rc = cwb_train_bernoulli_fused(c, Y, B, nu, M, offset_out, theta_agg_out, k_trace, sse_trace, risk_trace,
                                           s, &launched);
        if (rc || launched) return rc;
        if (c->path == 1)
            return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_train_bernoulli: fused path needs more shared memory than a CTA has");
    }
    return cwb_train_bernoulli_general(c, Y, B, nu, M, offset_out, theta_agg_out, k_trace, sse_trace, risk_trace, s);
}

int cwb_train_folds(cwb_ctx* c, const double* Y, int32_t B, const uint8_t* fold_of_row, int32_t F,
                    const int32_t* fold_of_rep, double nu, int32_t M, double* offset_out, double* theta_agg_out,
                    int32_t* k_trace, double* sse_trace, double* risk_trace, double* val_risk_trace, cudaStream_t s) {
    if (!c || !Y || !fold_of_row || !fold_of_rep || !theta_agg_out || B < 1 || M < 0 || F < 1 || F > 255 ||
        !(nu >= 0.0) || !isfinite(nu))
        return cwb_set_error(c, CWB_EINVAL, "cwb_train_folds: invalid argument");
    if (c->status) return c->status;
    c->stream = s;
    if (c->rows) return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_train_folds: row-sharded context");
    if (c->lshard) return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_train_folds: learner-sharded context");
    if (c->path == 3) return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_train_folds: the cross-Gram path (3) is cwb_train only");
    if (c->nb) return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_train_folds: unbinned pool (cwb_train only)");
    return cwb_train_folds_general(c, Y, B, fold_of_row, F, fold_of_rep, nu, M, offset_out, theta_agg_out, k_trace,
                                   sse_trace, risk_trace, val_risk_trace, s);
}

int cwb_train_acwb(cwb_ctx* c, const double* Y, int32_t B, double nu, double gamma, int32_t M,
                   double* offset_out, double* theta_f_out, double* theta_h_out, int32_t* k_trace,
                   int32_t* kcor_trace, double* sse_trace, double* risk_trace, cudaStream_t s) {
    if (!c || !Y || !theta_f_out || !theta_h_out || B < 1 || M < 0 || !(nu >= 0.0) || !isfinite(nu) ||
        !(gamma >= 0.0) || !isfinite(gamma))
        return cwb_set_error(c, CWB_EINVAL, "cwb_train_acwb: invalid argument");
    if (c->status) return c->status;
    c->stream = s;
    if (c->rows) return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_train_acwb: row-sharded context");
    if (c->lshard) return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_train_acwb: learner-sharded context");
    if (c->path == 3) return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_train_acwb: the cross-Gram path (3) is cwb_train only");
    if (c->nb) return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_train_acwb: unbinned pool (cwb_train only)");
    if (c->path != 2) {
        bool launched = false;
        int rc = cwb_train_acwb_fused(c, Y, B, nu, gamma, M, offset_out, theta_f_out, theta_h_out, k_trace,
                                      kcor_trace, sse_trace, risk_trace, s, &launched);
        if (rc || launched) return rc;
        if (c->path == 1)
            return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_train_acwb: fused path needs more shared memory than a CTA has");
    }
    return cwb_train_acwb_general(c, Y, B, nu, gamma, M, offset_out, theta_f_out, theta_h_out, k_trace, kcor_trace,
                                  sse_trace, risk_trace, s);
}

int cwb_train_hcwb(cwb_ctx* c, const double* Y, int32_t B, const uint8_t* val_mask, double nu, double gamma,
                   int32_t pat0, int32_t M, double* offset_out, double* theta_f_out, int32_t* k_trace,
                   int32_t* kcor_trace, double* sse_trace, double* risk_trace, double* val_risk_trace,
                   int32_t* switch_iter, cudaStream_t s) {
    if (!c || !Y || !val_mask || !theta_f_out || B < 1 || M < 0 || pat0 < 1 || !(nu >= 0.0) || !isfinite(nu) ||
        !(gamma >= 0.0) || !isfinite(gamma))
        return cwb_set_error(c, CWB_EINVAL, "cwb_train_hcwb: invalid argument");
    if (c->status) return c->status;
    c->stream = s;
    if (c->rows) return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_train_hcwb: row-sharded context");
    if (c->lshard) return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_train_hcwb: learner-sharded context");
    if (c->path == 3) return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_train_hcwb: the cross-Gram path (3) is cwb_train only");
    if (c->nb) return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_train_hcwb: unbinned pool (cwb_train only)");
    return cwb_train_hcwb_general(c, Y, B, val_mask, nu, gamma, pat0, M, offset_out, theta_f_out, k_trace, kcor_trace,
                                  sse_trace, risk_trace, val_risk_trace, switch_iter, s);
}

int cwb_fit_host(const double* X, int64_t n, int32_t K, const cwb_config* cfg, const double* Y, int32_t B,
                 double nu, int32_t M, double* offset_out, double* theta_agg_out, int32_t* k_trace,
                 double* sse_trace, double* risk_trace, cudaStream_t s) {
    if (!X || !Y || !theta_agg_out || n < 2 || K < 1 || B < 1 || M < 0)
        return cwb_set_error(nullptr, CWB_EINVAL, "cwb_fit_host: invalid argument");
    int d = (cfg ? cfg->n_knots + cfg->degree + 1 : 24);
    double *dX = nullptr, *dY = nullptr, *dOff = nullptr, *dAgg = nullptr, *dS = nullptr, *dR = nullptr;
    int32_t* dK = nullptr;
    const size_t mb = (size_t)M * B;
    bool ok = cwb_alloc((void**)&dX, 8 * (size_t)K * n, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&dY, 8 * (size_t)B * n, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&dOff, 8 * (size_t)B, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&dAgg, 8 * (size_t)B * K * d, s) == cudaSuccess;
    if (k_trace) ok &= cwb_alloc((void**)&dK, 4 * mb, s) == cudaSuccess;
    if (sse_trace) ok &= cwb_alloc((void**)&dS, 8 * mb, s) == cudaSuccess;
    if (risk_trace) ok &= cwb_alloc((void**)&dR, 8 * mb, s) == cudaSuccess;
    int rc = ok ? CWB_OK : cwb_set_error(nullptr, CWB_ENOMEM, "cwb_fit_host: allocation failed");
    cwb_ctx* c = nullptr;
    if (rc == CWB_OK) {
        cudaMemcpyAsync(dX, X, 8 * (size_t)K * n, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(dY, Y, 8 * (size_t)B * n, cudaMemcpyHostToDevice, s);
        rc = cwb_init(&c, dX, n, K, cfg, s);
    }
    if (rc == CWB_OK) rc = cwb_train(c, dY, B, nu, M, dOff, dAgg, dK, dS, dR, s);
    if (rc == CWB_OK) {
        if (offset_out) cudaMemcpyAsync(offset_out, dOff, 8 * (size_t)B, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(theta_agg_out, dAgg, 8 * (size_t)B * K * d, cudaMemcpyDeviceToHost, s);
        if (k_trace) cudaMemcpyAsync(k_trace, dK, 4 * mb, cudaMemcpyDeviceToHost, s);
        if (sse_trace) cudaMemcpyAsync(sse_trace, dS, 8 * mb, cudaMemcpyDeviceToHost, s);
        if (risk_trace) cudaMemcpyAsync(risk_trace, dR, 8 * mb, cudaMemcpyDeviceToHost, s);
        rc = cwb_status(c);
    }
    if (rc && c) g_err = c->err;  // the context's message outlives cwb_free
    if (c) cwb_free(c);
    cwb_release(dX, s); cwb_release(dY, s); cwb_release(dOff, s); cwb_release(dAgg, s);
    cwb_release(dK, s); cwb_release(dS, s); cwb_release(dR, s);
    if (rc == CWB_OK && cudaStreamSynchronize(s) != cudaSuccess)
        rc = cwb_set_error(nullptr, CWB_ECUDA, "cwb_fit_host: synchronisation failed");
    return rc;
}

int cwb_predict(cwb_ctx* c, const double* Xnew, int64_t m, const double* offset, const double* theta_agg,
                int32_t B, double* out, cudaStream_t s) {
    if (!c || !Xnew || !offset || !theta_agg || !out || m < 1 || B < 1)
        return cwb_set_error(c, CWB_EINVAL, "cwb_predict: invalid argument");
    if (c->status) return c->status;
    c->stream = s;
    if (c->nb) return cwb_nb_predict(c, Xnew, m, offset, theta_agg, B, out, s);
    return cwb_predict_impl(c, Xnew, m, offset, theta_agg, B, out, s);
}

int64_t cwb_launch_count(const cwb_ctx* c) { return c ? c->launches : 0; }

int cwb_set_h1_timing(cwb_ctx* c, int32_t on) {
    if (!c) return cwb_set_error(nullptr, CWB_EINVAL, "cwb_set_h1_timing: NULL context");
    c->h1_timing = on != 0;
    c->h1_ev_used = 0;
    return CWB_OK;
}

int cwb_get_h1_time(cwb_ctx* c, double* ms_total, int32_t* n_phases) {
    if (!c || !ms_total) return cwb_set_error(c, CWB_EINVAL, "cwb_get_h1_time: invalid argument");
    double t = 0.0;
    const int np = c->h1_ev_used / 2;
    if (np) {
        if (cudaEventSynchronize(c->h1_ev[2 * np - 1]) != cudaSuccess)
            return cwb_set_error(c, CWB_ECUDA, "cwb_get_h1_time: event synchronisation failed");
        for (int i = 0; i < np; i++) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, c->h1_ev[2 * i], c->h1_ev[2 * i + 1]) != cudaSuccess)
                return cwb_set_error(c, CWB_ECUDA, "cwb_get_h1_time: elapsed time");
            t += ms;
        }
    }
    *ms_total = t;
    if (n_phases) *n_phases = np;
    c->h1_ev_used = 0;
    return CWB_OK;
}

int cwb_set_phase_timing(cwb_ctx* c, int64_t* cycles4) {
    if (!c) return cwb_set_error(nullptr, CWB_EINVAL, "cwb_set_phase_timing: NULL context");
    c->timing = reinterpret_cast<long long*>(cycles4);
    return CWB_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ predict
namespace {
__global__ void k_pred_bins(const double* __restrict__ Xnew, int64_t m, int ns,
                            const double* __restrict__ bnd, int32_t* __restrict__ lix, int* status) {
    const int k = blockIdx.y;
    const double* bk = bnd + (size_t)k * (ns - 1);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        double v = Xnew[(size_t)k * m + i];
        if (!isfinite(v)) cwb_dev_fail(status, CWB_ENONFINITE);
        int a = 0, b = ns - 1;
        while (a < b) {
            int mid = a + ((b - a) >> 1);
            if (v <= bk[mid]) b = mid;
            else a = mid + 1;
        }
        lix[(size_t)k * m + i] = a;
    }
}

__global__ void k_pred_sum(const int32_t* __restrict__ lix, int64_t m, int K, int ns, int d,
                           const double* __restrict__ Zb, const double* __restrict__ offset,
                           const double* __restrict__ agg, double* __restrict__ out) {
    const int b = blockIdx.y;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        double v = offset[b];
        for (int k = 0; k < K; k++) {
            const double* zr = Zb + ((size_t)k * ns + lix[(size_t)k * m + i]) * d;
            const double* th = agg + ((size_t)b * K + k) * d;
            for (int j = 0; j < d; j++) v += zr[j] * th[j];
        }
        out[(size_t)b * m + i] = v;
    }
}
}  // namespace

int cwb_predict_impl(cwb_ctx* c, const double* Xnew, int64_t m, const double* offset,
                     const double* theta_agg, int32_t B, double* out, cudaStream_t s) {
    int32_t* lix = nullptr;
    if (cwb_alloc((void**)&lix, sizeof(int32_t) * (size_t)c->K * m, s) != cudaSuccess)
        return cwb_set_error(c, CWB_ENOMEM, "cwb_predict: allocation failed");
    unsigned gx = (unsigned)std::min<int64_t>(1184, (m + 255) / 256);
    k_pred_bins<<<dim3(gx, c->K), 256, 0, s>>>(Xnew, m, c->n_star, c->bnd, lix, c->d_status);
    k_pred_sum<<<dim3(gx, B), 256, 0, s>>>(lix, m, c->K, c->n_star, c->d, c->Zb, offset, theta_agg, out);
    c->launches += 2;
    cwb_release(lix, s);
    return cwb_check_launch(c, "predict kernels");
}
