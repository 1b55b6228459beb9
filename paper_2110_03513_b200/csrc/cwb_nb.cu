// cwb_nb.cu -- unbinned ("nb") base learners: the P-spline learner on
// the raw feature values, the setting binning is compared against (P:L842-846, P:L865,
// P:L1054).  Per row, a cubic B-spline basis on equidistant knots has 4 non-zero values
// at the knot span of x; the binMatVec scatter of the binned path becomes a
// 4-tap scatter into the d coefficient slots:
//
//   init    span s_k(i) = knot interval of x_ki (u8), t = (x - knot_s) / h in [0, 1];
//           rows of every learner grouped by span (the bin inversion kernel k_csr with
//           the spans as "bins"); G_k = Z_k^T Z_k from per-span 4 x 4 blocks; then
//           df -> lambda and the cached inverse as for the binned pool (k_lambda).
//   H1+H2   s_k[j][b] = sum_i B_j(x_ki) r_i[b]: warp per (learner, span, chunk of the
//           span's rows), lane = replication column, 4 accumulators; the chunk partials
//           are added in (span, chunk) order by k_nb_comb (deterministic).
//   H3-H5   k_h234 (from s) and k_h5 of the general path.
//   H6      r_i -= nu sum_t B_{s+t}(x_{k* i}) theta*_{s+t}, r^T r partials.
//
// Values of the uniform cubic B-spline at t (Cox-de Boor on equidistant knots, closed
// form): (1-t)^3/6, (3t^3 - 6t^2 + 4)/6, (-3t^3 + 3t^2 + 3t + 1)/6, t^3/6 for the basis
// functions s, s+1, s+2, s+3 (0-based, knots t_q = lo + (q - 3) h as in the binned pool).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "cwb_internal.cuh"

namespace {

constexpr int kCH = 1024;  // rows per H12 work item

__device__ __forceinline__ void cubic4(double t, double v[4]) {
    const double u = 1.0 - t, t2 = t * t, t3 = t2 * t;
    v[0] = u * u * u / 6.0;
    v[1] = (3.0 * t3 - 6.0 * t2 + 4.0) / 6.0;
    v[2] = (-3.0 * t3 + 3.0 * t2 + 3.0 * t + 1.0) / 6.0;
    v[3] = t3 / 6.0;
}

// span and position of every (k, i): s = clamp(floor((x - lo) / h), 0, S - 1)
__global__ void k_nb_span(const double* __restrict__ X, int64_t n, const double* __restrict__ lo,
                          const double* __restrict__ hi, int S, uint8_t* __restrict__ sp, double* __restrict__ tn) {
    const int k = blockIdx.y;
    const double l = lo[k], h = (hi[k] - l) / (double)S;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double x = X[(size_t)k * n + i];
        int s = (int)floor((x - l) / h);
        s = max(0, min(S - 1, s));
        const double kn = l + (double)s * h;
        sp[(size_t)k * n + i] = (uint8_t)s;
        tn[(size_t)k * n + i] = (x - kn) / h;
    }
}

// t in span-sorted order
template <typename PermT>
__global__ void k_nb_sort_t(const double* __restrict__ tn, const PermT* __restrict__ perm, int64_t n,
                            double* __restrict__ ts) {
    const int k = blockIdx.y;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        ts[(size_t)k * n + j] = tn[(size_t)k * n + (uint32_t)perm[(size_t)k * n + j]];
}

// per (span s, learner k): the 10 products v_a v_b (a <= b) summed over the span's rows
__global__ void k_nb_gram_part(const double* __restrict__ ts, const int32_t* __restrict__ off, int64_t n, int S,
                               double* __restrict__ Gs) {
    const int s = blockIdx.x, k = blockIdx.y;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int32_t a0 = off[(size_t)k * (S + 1) + s], a1 = off[(size_t)k * (S + 1) + s + 1];
    double acc[10];
#pragma unroll
    for (int e = 0; e < 10; e++) acc[e] = 0.0;
    for (int32_t j = a0 + threadIdx.x; j < a1; j += blockDim.x) {
        double v[4];
        cubic4(ts[(size_t)k * n + j], v);
        int e = 0;
#pragma unroll
        for (int a = 0; a < 4; a++)
#pragma unroll
            for (int b = a; b < 4; b++) acc[e++] += v[a] * v[b];
    }
    __shared__ double red[10][32];
#pragma unroll
    for (int e = 0; e < 10; e++) {
        const double t = warp_sum(acc[e]);
        if (lane == 0) red[e][w] = t;
    }
    __syncthreads();
    if (threadIdx.x < 10) {
        double t = 0.0;
        for (int q = 0; q < nw; q++) t += red[threadIdx.x][q];
        Gs[((size_t)k * S + s) * 10 + threadIdx.x] = t;
    }
}

__device__ __forceinline__ int pair10(int a, int b) {  // a <= b < 4 -> 0..9 in the order of k_nb_gram_part
    return a * 4 - a * (a - 1) / 2 + (b - a);
}

// G_k[j][j'] = sum over spans s (ascending) with s <= min(j, j'), max(j, j') <= s + 3
__global__ void k_nb_gram_fin(const double* __restrict__ Gs, int S, int d, double* __restrict__ G) {
    const int k = blockIdx.x;
    for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
        const int j = e / d, jp = e - j * d;
        const int a = min(j, jp), b = max(j, jp);
        double v = 0.0;
        for (int s = max(0, b - 3); s <= min(S - 1, a); s++) v += Gs[((size_t)k * S + s) * 10 + pair10(a - s, b - s)];
        G[(size_t)k * d * d + e] = v;
    }
}

// item q of learner k -> (span, chunk); false when q is past the last chunk
__device__ __forceinline__ bool nb_item(const uint32_t* __restrict__ cnt, int k, int S, int q, int& s, int& ch) {
    for (s = 0; s < S; s++) {
        const int nc = (int)((cnt[(size_t)k * S + s] + kCH - 1) / kCH);
        if (q < nc) { ch = q; return true; }
        q -= nc;
    }
    return false;
}

// H1+H2: warp per (learner k, item q), lane = column b: P[k][q][t][b] = sum over the item's rows
// of B_{s+t}(x_i) r_i[b]
template <typename PermT>
__global__ void k_h12_nb(const double* __restrict__ Rt, int64_t n, int Bp, int K, int S, int Q,
                         const uint32_t* __restrict__ cnt, const int32_t* __restrict__ off,
                         const PermT* __restrict__ perm, const double* __restrict__ ts, double* __restrict__ P) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + w;
    if (g >= (int64_t)K * Q) return;
    const int k = (int)(g / Q), q = (int)(g - (int64_t)k * Q);
    int s, ch;
    if (!nb_item(cnt, k, S, q, s, ch)) return;
    const int b = blockIdx.y * 32 + lane;
    const int32_t a0 = off[(size_t)k * (S + 1) + s] + ch * kCH;
    const int32_t a1 = min(off[(size_t)k * (S + 1) + s + 1], a0 + kCH);
    const PermT* pk = perm + (size_t)k * n;
    const double* tk = ts + (size_t)k * n;
    const double* col = Rt + b;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    int32_t j = a0;
    for (; j + 2 <= a1; j += 2) {
        const uint32_t i0 = pk[j], i1 = pk[j + 1];
        const double r0 = col[(size_t)i0 * Bp], r1 = col[(size_t)i1 * Bp];
        double v0[4], v1[4];
        cubic4(tk[j], v0);
        cubic4(tk[j + 1], v1);
#pragma unroll
        for (int t = 0; t < 4; t++) {
            acc[t] += v0[t] * r0;
            acc[t] += v1[t] * r1;
        }
    }
    if (j < a1) {
        const double r0 = col[(size_t)pk[j] * Bp];
        double v0[4];
        cubic4(tk[j], v0);
#pragma unroll
        for (int t = 0; t < 4; t++) acc[t] += v0[t] * r0;
    }
#pragma unroll
    for (int t = 0; t < 4; t++) P[(((size_t)k * Q + q) * 4 + t) * Bp + b] = acc[t];
}

// Sg[k][j][b] = sum over spans s = j-3..j (ascending), chunks ascending, of P[k][q][j - s][b]
__global__ void k_nb_comb(const double* __restrict__ P, int Bp, int K, int S, int Q, int d,
                          const uint32_t* __restrict__ cnt, double* __restrict__ Sg) {
    const int k = blockIdx.x / d, j = blockIdx.x - (blockIdx.x / d) * d;
    const int b = blockIdx.y * blockDim.x + threadIdx.x;
    if (b >= Bp) return;
    double v = 0.0;
    int q0 = 0;
    for (int s = 0; s < S; s++) {
        const int nc = (int)((cnt[(size_t)k * S + s] + kCH - 1) / kCH);
        if (s >= j - 3 && s <= j)
            for (int c = 0; c < nc; c++) v += P[(((size_t)k * Q + q0 + c) * 4 + (j - s)) * Bp + b];
        q0 += nc;
    }
    Sg[((size_t)k * d + j) * Bp + b] = v;
}

// H6: r_i -= nu sum_t B_{s+t}(x_{k* i}) theta*_{s+t} for column b's learner k*, r^T r partials
__global__ void k_h6_nb(double* __restrict__ Rt, int64_t n, int Bp, int d, const int32_t* __restrict__ kstar,
                        const uint8_t* __restrict__ sp, const double* __restrict__ tn, const double* __restrict__ theta,
                        double nu, int rows_per_blk, double* __restrict__ part) {
    __shared__ double red[8][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int b = blockIdx.y * 32 + lane;
    const int ks = kstar[b];
    const uint8_t* spk = sp + (size_t)ks * n;
    const double* tk = tn + (size_t)ks * n;
    const double* th = theta + (size_t)ks * d * Bp + b;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_blk;
    const int64_t r1 = min(n, r0 + rows_per_blk);
    double acc = 0.0;
    for (int64_t i = r0 + w; i < r1; i += 8) {
        const int s = spk[i];
        double v[4];
        cubic4(tk[i], v);
        double z = 0.0;
#pragma unroll
        for (int t = 0; t < 4; t++) z += v[t] * th[(size_t)(s + t) * Bp];
        const double r = Rt[(size_t)i * Bp + b] - nu * z;
        Rt[(size_t)i * Bp + b] = r;
        acc += r * r;
    }
    red[w][lane] = acc;
    __syncthreads();
    if (w == 0) {
        double t = 0.0;
        for (int q = 0; q < 8; q++) t += red[q][lane];
        part[(size_t)blockIdx.x * Bp + b] = t;
    }
}

// prediction with unbinned learners: out[b][i] = offset[b] + sum_k sum_t B_{s+t}(x) theta_agg[b][k][s+t],
// x = Xnew[k][i] clamped to [lo_k, hi_k] (reading U2)
__global__ void k_pred_nb(const double* __restrict__ Xnew, int64_t m, int K, int d, int S,
                          const double* __restrict__ lo, const double* __restrict__ hi,
                          const double* __restrict__ offset, const double* __restrict__ agg, double* __restrict__ out,
                          int* status) {
    const int b = blockIdx.y;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        double v = offset[b];
        for (int k = 0; k < K; k++) {
            double x = Xnew[(size_t)k * m + i];
            if (!isfinite(x)) cwb_dev_fail(status, CWB_ENONFINITE);
            const double l = lo[k], h = (hi[k] - l) / (double)S;
            x = fmin(fmax(x, l), hi[k]);
            int s = (int)floor((x - l) / h);
            s = max(0, min(S - 1, s));
            double bv[4];
            cubic4((x - (l + (double)s * h)) / h, bv);
            const double* th = agg + ((size_t)b * K + k) * d + s;
#pragma unroll
            for (int t = 0; t < 4; t++) v += bv[t] * th[t];
        }
        out[(size_t)b * m + i] = v;
    }
}

}  // namespace

int cwb_nb_predict(cwb_ctx* c, const double* Xnew, int64_t m, const double* offset, const double* theta_agg,
                   int32_t B, double* out, cudaStream_t s) {
    const unsigned gx = (unsigned)std::min<int64_t>(1184, (m + 255) / 256);
    k_pred_nb<<<dim3(gx, B), 256, 0, s>>>(Xnew, m, c->K, c->d, c->nb_spans, c->lo, c->hi, offset, theta_agg, out,
                                          c->d_status);
    c->launches += 1;
    return cwb_check_launch(c, "unbinned predict kernel");
}

// ===================================================================== host

void cwb_nb_release(cwb_ctx* c, cudaStream_t s) {
    cwb_release(c->nb_sp, s); cwb_release(c->nb_t, s); cwb_release(c->nb_ts, s); cwb_release(c->nb_cnt, s);
    cwb_release(c->nb_off, s); cwb_release(c->nb_perm, s); cwb_release(c->nb_P, s); cwb_release(c->nb_S, s);
    c->nb_sp = nullptr; c->nb_t = c->nb_ts = c->nb_P = c->nb_S = nullptr;
    c->nb_cnt = nullptr; c->nb_off = nullptr; c->nb_perm = nullptr; c->nb_Pbytes = 0;
}

// Unbinned pool tables and G (replaces the binned G before k_lambda).
int cwb_nb_init(cwb_ctx* c, const double* X, cudaStream_t s) {
    const int K = c->K, S = c->n_knots + 1, d = c->d;
    const int64_t n = c->n;
    c->nb_spans = S;
    c->nb_Q = (int32_t)((n + kCH - 1) / kCH) + S;
    bool ok = true;
    ok &= cwb_alloc((void**)&c->nb_sp, (size_t)K * n + 16, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&c->nb_t, sizeof(double) * K * n, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&c->nb_ts, sizeof(double) * K * n, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&c->nb_cnt, sizeof(uint32_t) * K * S, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&c->nb_off, sizeof(int32_t) * K * (S + 1), s) == cudaSuccess;
    ok &= cwb_alloc(&c->nb_perm, (size_t)c->perm_bytes * ((size_t)K * n + 8), s) == cudaSuccess;
    double* Gs = nullptr;
    ok &= cwb_alloc((void**)&Gs, sizeof(double) * K * S * 10, s) == cudaSuccess;
    if (!ok) {
        cwb_release(Gs, s);
        return cwb_set_error(c, CWB_ENOMEM, "unbinned pool allocation failed");
    }
    const int gx = (int)std::min<int64_t>(1184, (n + 255) / 256);
    k_nb_span<<<dim3(gx, K), 256, 0, s>>>(X, n, c->lo, c->hi, S, c->nb_sp, c->nb_t);
    int rc = cwb_launch_csr(c, c->nb_sp, 1, n, K, S, c->nb_cnt, c->nb_off, c->nb_perm, c->perm_bytes, s);
    if (rc) { cwb_release(Gs, s); return rc; }
    if (c->perm_bytes == 2)
        k_nb_sort_t<uint16_t><<<dim3(gx, K), 256, 0, s>>>(c->nb_t, (const uint16_t*)c->nb_perm, n, c->nb_ts);
    else
        k_nb_sort_t<uint32_t><<<dim3(gx, K), 256, 0, s>>>(c->nb_t, (const uint32_t*)c->nb_perm, n, c->nb_ts);
    k_nb_gram_part<<<dim3(S, K), 256, 0, s>>>(c->nb_ts, c->nb_off, n, S, Gs);
    k_nb_gram_fin<<<K, 256, 0, s>>>(Gs, S, d, c->G);
    c->launches += 4;
    cwb_release(Gs, s);
    return cwb_check_launch(c, "unbinned pool kernels");
}

// H1 + H2 of the unbinned pool for the residual columns of Rt: s into Sg[K][d][Bp]
int cwb_nb_h12(cwb_ctx* c, const double* Rt, int Bp, double* Sg, cudaStream_t s) {
    const int K = c->K, S = c->nb_spans, Q = c->nb_Q, d = c->d;
    const size_t need = sizeof(double) * (size_t)K * Q * 4 * Bp;
    if (c->nb_Pbytes < need) {
        cwb_release(c->nb_P, s);
        c->nb_P = nullptr;
        c->nb_Pbytes = 0;
        if (cwb_alloc((void**)&c->nb_P, need, s) != cudaSuccess)
            return cwb_set_error(c, CWB_ENOMEM, "unbinned H12 workspace allocation failed");
        c->nb_Pbytes = need;
    }
    const int wpb = 8;
    dim3 grid((unsigned)(((int64_t)K * Q + wpb - 1) / wpb), Bp / 32);
    if (c->perm_bytes == 2)
        k_h12_nb<uint16_t><<<grid, wpb * 32, 0, s>>>(Rt, c->n, Bp, K, S, Q, c->nb_cnt, c->nb_off,
                                                    (const uint16_t*)c->nb_perm, c->nb_ts, c->nb_P);
    else
        k_h12_nb<uint32_t><<<grid, wpb * 32, 0, s>>>(Rt, c->n, Bp, K, S, Q, c->nb_cnt, c->nb_off,
                                                    (const uint32_t*)c->nb_perm, c->nb_ts, c->nb_P);
    k_nb_comb<<<dim3(K * d, (Bp + 31) / 32), 32, 0, s>>>(c->nb_P, Bp, K, S, Q, d, c->nb_cnt, Sg);
    c->launches += 2;
    return CWB_OK;
}

// H6 of the unbinned pool (theta of every learner in theta[K][d][Bp], k* per column)
void cwb_nb_h6(cwb_ctx* c, double* Rt, int Bp, const int32_t* kstar, const double* theta, double nu,
               int rows_per_blk, int nblk, double* part, cudaStream_t s) {
    k_h6_nb<<<dim3(nblk, Bp / 32), 256, 0, s>>>(Rt, c->n, Bp, c->d, kstar, c->nb_sp, c->nb_t, theta, nu,
                                                rows_per_blk, part);
    c->launches += 1;
}
