// cwb_init.cu -- one-off pool construction on the device (I1-I7).
//
//   I1 k_minmax   per-learner min / max of x
//   I2 k_design   design points z and bin boundaries
//   I3 k_bin      index vector (binary search on the boundaries)
//   I4 k_csr      bin inversion: rows of every bin, ascending      (binning as a hash map)
//   I5 k_basis    cubic B-spline basis at the design points
//   I6 k_gram     G = Zb^T diag(cnt) Zb  (binMatMat, w = 1)
//   I7 k_dro      Demmler-Reinsch df -> lambda, (G + lambda D)^-1  supp. P:L314-319
//
// Everything here runs once per data set and is shared by all B
// replications.  Bit-exactness with the paper's fp64 definitions matters for
// I2/I3 (integer bin decisions): they use explicit round-to-nearest
// intrinsics so that no FMA contraction changes a rounding.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "cwb_internal.cuh"

namespace {

// ---------------------------------------------------------------- I1 min/max
__global__ void k_minmax(const double* __restrict__ X, int64_t n, double* lo, double* hi,
                         int* status) {
    const int k = blockIdx.x;
    const double* x = X + (size_t)k * n;
    double mn = INFINITY, mx = -INFINITY;
    bool bad = false;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        double v = x[i];
        bad |= !isfinite(v);
        mn = fmin(mn, v);
        mx = fmax(mx, v);
    }
    __shared__ double smn[32], smx[32];
    __shared__ int sbad;
    if (threadIdx.x == 0) sbad = 0;
    __syncthreads();
    if (bad) atomicOr(&sbad, 1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) { smn[w] = mn; smx[w] = mx; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < nw; i++) { mn = fmin(mn, smn[i]); mx = fmax(mx, smx[i]); }
        lo[k] = mn;
        hi[k] = mx;
        if (sbad) cwb_dev_fail(status, CWB_ENONFINITE);
        else if (!(mn < mx)) cwb_dev_fail(status, CWB_EDEGENERATE);
    }
}

// z_l = lo + (l/(n*-1)) (hi - lo), z_{n*-1} = hi, each operation rounded once
__device__ __forceinline__ double design_point(double lo, double hi, int l, int ns) {
    if (l == ns - 1) return hi;
    double t = __ddiv_rn((double)l, (double)(ns - 1));
    return __dadd_rn(lo, __dmul_rn(t, __dsub_rn(hi, lo)));
}

// ---------------------------------------------------------- I2 design points
__global__ void k_design(const double* lo_, const double* hi_, int ns, double* z, double* bnd,
                         const int* status) {
    if (status && *status) return;
    const int k = blockIdx.x;
    const double lo = lo_[k], hi = hi_[k];
    for (int l = threadIdx.x; l < ns; l += blockDim.x) {
        double zl = design_point(lo, hi, l, ns);
        z[(size_t)k * ns + l] = zl;
        if (l < ns - 1) {
            double zr = design_point(lo, hi, l + 1, ns);
            bnd[(size_t)k * (ns - 1) + l] = __dadd_rn(zl, __ddiv_rn(__dsub_rn(zr, zl), 2.0));
        }
    }
}

// ------------------------------------------------------------ I3 index vector
// idx(x) = smallest l with x <= bnd_l, else n*-1 (P:L861 closed-right bins).
template <typename IdxT, bool SMEM>
__global__ void k_bin(const double* __restrict__ X, int64_t n, int ns, const double* __restrict__ bnd,
                      IdxT* __restrict__ idx, const int* status) {
    extern __shared__ double sb[];
    if (status && *status) return;
    const int k = blockIdx.y;
    const double* bk = bnd + (size_t)k * (ns - 1);
    if (SMEM) {
        for (int l = threadIdx.x; l < ns - 1; l += blockDim.x) sb[l] = bk[l];
        __syncthreads();
    }
    const double* bs = SMEM ? sb : bk;
    const double* x = X + (size_t)k * n;
    IdxT* out = idx + (size_t)k * n;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double v = x[i];
        int a = 0, b = ns - 1;
        while (a < b) {
            int mid = a + ((b - a) >> 1);
            if (v <= bs[mid]) b = mid;
            else a = mid + 1;
        }
        out[i] = (IdxT)a;
    }
}

// --------------------------------------------------------- I4 bin inversion
// Stable counting sort of the rows by bin (per learner = blockIdx.x):
// cnt[l] = #rows in bin l, off[l] = first slot of bin l, perm[off[l]..] = rows
// of bin l in increasing order.  Each warp owns a contiguous row range; ranks
// inside a warp come from __match_any_sync, so the result is deterministic.
template <typename IdxT, typename PermT>
__global__ void k_csr(const IdxT* __restrict__ idx, int64_t n, int ns, int nw_use,
                      uint32_t* __restrict__ cnt_out, int32_t* __restrict__ off_out,
                      PermT* __restrict__ perm_out, const int* status) {
    extern __shared__ uint32_t sm[];
    if (status && *status) return;
    const int k = blockIdx.x;
    const IdxT* id = idx + (size_t)k * n;
    uint32_t* cntw = sm;                                  // nw_use x ns
    uint32_t* tot = sm + (size_t)nw_use * ns;             // ns
    __shared__ uint32_t wsum[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nthr = blockDim.x;
    for (int64_t a = threadIdx.x; a < (int64_t)nw_use * ns; a += nthr) cntw[a] = 0;
    __syncthreads();
    const int64_t L = (n + nw_use - 1) / nw_use;
    const int64_t r0 = (int64_t)w * L, r1 = min(n, r0 + L);
    if (w < nw_use)
        for (int64_t i = r0 + lane; i < r1; i += 32) atomicAdd(&cntw[(size_t)w * ns + id[i]], 1u);
    __syncthreads();
    // exclusive prefix over warps per bin, totals per bin
    for (int b = threadIdx.x; b < ns; b += nthr) {
        uint32_t run = 0;
        for (int q = 0; q < nw_use; q++) {
            uint32_t c = cntw[(size_t)q * ns + b];
            cntw[(size_t)q * ns + b] = run;
            run += c;
        }
        tot[b] = run;
        cnt_out[(size_t)k * ns + b] = run;
    }
    __syncthreads();
    // exclusive block scan of tot -> offsets (each thread: a contiguous chunk)
    const int per = (ns + nthr - 1) / nthr;
    const int b0 = threadIdx.x * per, b1 = min(ns, b0 + per);
    uint32_t local = 0;
    for (int b = b0; b < b1; b++) local += tot[b];
    uint32_t inc = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    if (w == 0) {
        uint32_t v = lane < (nthr >> 5) ? wsum[lane] : 0u;
        uint32_t s = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t t = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += t;
        }
        wsum[lane] = s - v;  // exclusive warp offsets
    }
    __syncthreads();
    uint32_t base = wsum[w] + inc - local;
    __syncthreads();
    int32_t* off = off_out + (size_t)k * (ns + 1);
    for (int b = b0; b < b1; b++) {
        uint32_t c = tot[b];
        tot[b] = base;  // tot now holds off[b]
        off[b] = (int32_t)base;
        base += c;
    }
    if (threadIdx.x == 0) off[ns] = (int32_t)n;
    __syncthreads();
    // per-warp base slot of every bin
    for (int64_t a = threadIdx.x; a < (int64_t)nw_use * ns; a += nthr) cntw[a] += tot[a % ns];
    __syncthreads();
    if (w < nw_use) {
        PermT* perm = perm_out + (size_t)k * n;
        uint32_t* mybase = cntw + (size_t)w * ns;
        for (int64_t s0 = r0; s0 < r1; s0 += 32) {
            int64_t i = s0 + lane;
            bool valid = i < r1;
            uint32_t b = valid ? (uint32_t)id[i] : 0xffffffffu;
            uint32_t mask = __match_any_sync(0xffffffffu, b);
            uint32_t lt = mask & ((1u << lane) - 1u);
            uint32_t slot = 0;
            if (valid) {
                slot = mybase[b] + __popc(lt);
                perm[slot] = (PermT)i;
            }
            __syncwarp();
            if (valid && lt == 0) mybase[b] += __popc(mask);
            __syncwarp();
        }
    }
}

// ------------------------------------------------------------------ I5 basis
// Local de Boor evaluation of the degree+1 non-zero B-splines at z on the
// knots t_q = lo + (q - degree) h, h = (hi - lo)/(n_knots + 1) (reading G6).
__device__ __forceinline__ double knot(double lo, double h, int q, int deg) {
    return __dadd_rn(lo, __dmul_rn((double)(q - deg), h));
}

__global__ void k_basis(const double* __restrict__ z, const double* lo_, const double* hi_, int ns,
                        int deg, int nk, int d, double* Zb, int32_t* zj0, double* Zs,
                        int32_t* lwin, const int* status) {
    extern __shared__ int32_t sj0[];
    if (status && *status) return;
    const int k = blockIdx.x;
    const double lo = lo_[k], hi = hi_[k];
    const double h = __ddiv_rn(__dsub_rn(hi, lo), (double)(nk + 1));
    const int ntk = nk + 2 * deg + 2;  // number of knots
    const int W4 = d < CWB_SPW ? d : CWB_SPW;
    for (int l = threadIdx.x; l < ns; l += blockDim.x) {
        const double x = z[(size_t)k * ns + l];
        // knot span s with t_s <= x < t_{s+1} (the degree-0 B-spline indicator)
        int s = deg + (int)floor((x - lo) / h);
        if (s < 0) s = 0;
        if (s > ntk - 2) s = ntk - 2;
        while (s > 0 && x < knot(lo, h, s, deg)) s--;
        while (s + 1 < ntk - 1 && x >= knot(lo, h, s + 1, deg)) s++;
        double N[CWB_SPW], left[CWB_SPW], right[CWB_SPW];
        N[0] = 1.0;
        for (int j = 1; j <= deg; j++) {
            left[j] = x - knot(lo, h, s + 1 - j, deg);
            right[j] = knot(lo, h, s + j, deg) - x;
            double saved = 0.0;
            for (int r = 0; r < j; r++) {
                double tmp = N[r] / (right[r + 1] + left[j - r]);
                N[r] = saved + right[r + 1] * tmp;
                saved = left[j - r] * tmp;
            }
            N[j] = saved;
        }
        // basis index of N[r] is s - deg + r; keep the window inside [0, d)
        int j0 = s - deg;
        int w0 = j0 < 0 ? 0 : j0;
        if (w0 > d - W4) w0 = d - W4;
        double* zrow = Zb + ((size_t)k * ns + l) * d;
        for (int j = 0; j < d; j++) zrow[j] = 0.0;
        double* srow = Zs + ((size_t)k * ns + l) * CWB_SPW;
        for (int q = 0; q < CWB_SPW; q++) {
            int j = w0 + q;
            int r = j - j0;
            double v = (q < W4 && r >= 0 && r <= deg && j < d) ? N[r] : 0.0;
            srow[q] = v;
            if (q < W4) zrow[j] = v;
        }
        zj0[(size_t)k * ns + l] = w0;
        sj0[l] = w0;
    }
    __syncthreads();
    // design-point window of basis j: l with j - 3 <= zj0[l] <= j (zj0 non-decreasing)
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
        int a = 0, b = ns;  // first l with zj0[l] >= j - (W4-1)
        while (a < b) { int m = (a + b) >> 1; if (sj0[m] >= j - (W4 - 1)) b = m; else a = m + 1; }
        int lb = a;
        a = lb; b = ns;     // first l with zj0[l] > j
        while (a < b) { int m = (a + b) >> 1; if (sj0[m] > j) b = m; else a = m + 1; }
        lwin[((size_t)k * d + j) * 2 + 0] = lb;
        lwin[((size_t)k * d + j) * 2 + 1] = a;
    }
}

// ---------------------------------------------------------- I6 binMatMat (G)
__global__ void k_gram(const double* __restrict__ Zb, const uint32_t* __restrict__ cnt, int ns, int d,
                       const int32_t* __restrict__ lwin, double* G, const int* status) {
    if (status && *status) return;
    const int k = blockIdx.x;
    for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
        const int a = e / d, b = e % d;
        double s = 0.0;
        if (abs(a - b) < CWB_SPW) {
            const int l0 = max(lwin[((size_t)k * d + a) * 2], lwin[((size_t)k * d + b) * 2]);
            const int l1 = min(lwin[((size_t)k * d + a) * 2 + 1], lwin[((size_t)k * d + b) * 2 + 1]);
            for (int l = l0; l < l1; l++) {
                const double* zr = Zb + ((size_t)k * ns + l) * d;
                s += (double)cnt[(size_t)k * ns + l] * (zr[a] * zr[b]);
            }
        }
        G[((size_t)k * d + a) * d + b] = s;
    }
}

// --------------------------------------------------- I7 DRO, lambda, inverse
#define DS 33  // padded shared row stride

__device__ void blk_cholesky(double (*P)[DS], int d, int* fail) {
    // in place: lower triangle of P becomes L with P = L L^T
    for (int j = 0; j < d; j++) {
        if (threadIdx.x == 0) {
            double v = P[j][j];
            if (!(v > 0.0)) *fail = 1;
            P[j][j] = sqrt(fmax(v, 1e-300));
        }
        __syncthreads();
        for (int i = j + 1 + threadIdx.x; i < d; i += blockDim.x) P[i][j] /= P[j][j];
        __syncthreads();
        for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
            const int i = e / d, c = e % d;
            if (c > j && i >= c) P[i][c] -= P[i][j] * P[c][j];
        }
        __syncthreads();
    }
}

__device__ void blk_tri_inverse(double (*L)[DS], double (*W)[DS], int d) {
    // W = L^{-1} (lower triangular), one column per thread
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        for (int i = 0; i < d; i++) {
            if (i < c) { W[i][c] = 0.0; continue; }
            double s = (i == c) ? 1.0 : 0.0;
            for (int q = c; q < i; q++) s -= L[i][q] * W[q][c];
            W[i][c] = s / L[i][i];
        }
    }
    __syncthreads();
}

__device__ __forceinline__ double df_term(double mu, double lam, int kind) {
    // eigenvalue of the hat matrix in the DRO basis: h = mu / (mu + lam (1 - mu))
    double den = mu + lam * (1.0 - mu);
    if (!(den > 0.0)) return 0.0;
    double h = mu / den;
    return kind == 2 ? h * (2.0 - h) : h;
}

__global__ void k_dro(const double* __restrict__ Gall, int d, double target, int kind,
                      double* lambda_out, double* Ainv_out, double* eig_out, int* status) {
    __shared__ double G[CWB_MAX_D][DS], P[CWB_MAX_D][DS], W[CWB_MAX_D][DS], T[CWB_MAX_D][DS];
    __shared__ double cs[CWB_MAX_D / 2][2];
    __shared__ int pq[CWB_MAX_D / 2][2];
    __shared__ int fail;
    __shared__ double s_lambda, s_off;
    if (status && *status) return;
    const int k = blockIdx.x;
    const int tid = threadIdx.x, nthr = blockDim.x;
    if (tid == 0) fail = 0;
    for (int e = tid; e < d * d; e += nthr) {
        const int a = e / d, b = e % d;
        const double g = Gall[((size_t)k * d + a) * d + b];
        // D = Delta^T Delta, Delta rows (.., 1, -2, 1, ..)  (supp. P:L312)
        double dv = 0.0;
        for (int i = 0; i + 2 < d; i++) {
            double ca = (a == i) ? 1.0 : (a == i + 1) ? -2.0 : (a == i + 2) ? 1.0 : 0.0;
            double cb = (b == i) ? 1.0 : (b == i + 1) ? -2.0 : (b == i + 2) ? 1.0 : 0.0;
            dv += ca * cb;
        }
        G[a][b] = g;
        T[a][b] = dv;          // keep D in T until it is needed again
        P[a][b] = g + dv;      // whitening matrix G + D (PD, reading G19)
    }
    __syncthreads();
    blk_cholesky(P, d, &fail);
    if (fail) { if (tid == 0) cwb_dev_fail(status, CWB_ECALIB); return; }
    blk_tri_inverse(P, W, d);  // W = R^{-1},  G + D = R R^T
    // M = W G W^T  (symmetric, eigenvalues mu in [0, 1])
    double (*Dm)[DS] = T;
    __shared__ double M[CWB_MAX_D][DS];
    for (int e = tid; e < d * d; e += nthr) {  // P <- W G
        const int i = e / d, c = e % d;
        double s = 0.0;
        for (int q = 0; q <= i; q++) s += W[i][q] * G[q][c];
        P[i][c] = s;
    }
    __syncthreads();
    for (int e = tid; e < d * d; e += nthr) {  // M <- (W G) W^T, lower half mirrored
        const int i = e / d, c = e % d;
        if (c <= i) {
            double s = 0.0;
            for (int q = 0; q <= c; q++) s += P[i][q] * W[c][q];
            M[i][c] = s;
            M[c][i] = s;
        }
    }
    __syncthreads();
    // cyclic parallel Jacobi (round-robin pairs; disjoint rotations commute)
    const int m = d + (d & 1);
    for (int sweep = 0; sweep < 40; sweep++) {
        if (tid < 32) {
            double o = 0.0;
            for (int e = tid; e < d * d; e += 32) { const int i = e / d, c = e % d; if (i != c) o += M[i][c] * M[i][c]; }
            o = warp_sum(o);
            if (tid == 0) s_off = o;
        }
        __syncthreads();
        if (s_off < 1e-34) break;
        for (int st = 0; st < m - 1; st++) {
            if (tid < m / 2) {
                int a0 = (tid == 0) ? 0 : 1 + ((tid - 1 + st) % (m - 1));
                int b0 = 1 + ((m - 1 - tid - 1 + st) % (m - 1));
                int p = min(a0, b0), q = max(a0, b0);
                double c = 1.0, s = 0.0;
                if (q < d && M[p][q] != 0.0) {
                    double tau = (M[q][q] - M[p][p]) / (2.0 * M[p][q]);
                    double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                    c = 1.0 / sqrt(1.0 + t * t);
                    s = t * c;
                }
                cs[tid][0] = c; cs[tid][1] = s;
                pq[tid][0] = p; pq[tid][1] = (q < d) ? q : -1;
            }
            __syncthreads();
            for (int e = tid; e < (m / 2) * d; e += nthr) {  // rows: M <- J^T M
                const int pr = e / d, j = e % d;
                const int p = pq[pr][0], q = pq[pr][1];
                if (q >= 0) {
                    const double c = cs[pr][0], s = cs[pr][1];
                    const double ap = M[p][j], aq = M[q][j];
                    M[p][j] = c * ap - s * aq;
                    M[q][j] = s * ap + c * aq;
                }
            }
            __syncthreads();
            for (int e = tid; e < (m / 2) * d; e += nthr) {  // columns: M <- M J
                const int pr = e / d, j = e % d;
                const int p = pq[pr][0], q = pq[pr][1];
                if (q >= 0) {
                    const double c = cs[pr][0], s = cs[pr][1];
                    const double ap = M[j][p], aq = M[j][q];
                    M[j][p] = c * ap - s * aq;
                    M[j][q] = s * ap + c * aq;
                }
            }
            __syncthreads();
        }
    }
    // lambda: df(lambda) = target, bisection on log2(lambda) (df decreasing)
    if (tid < 32) {
        double mu = 0.0;
        if (tid < d) mu = fmin(1.0, fmax(0.0, M[tid][tid]));
        if (tid < d) eig_out[(size_t)k * d + tid] = mu;
        double elo = -150.0, ehi = 150.0;
        double dlo = warp_sum(tid < d ? df_term(mu, exp2(elo), kind) : 0.0);
        double dhi = warp_sum(tid < d ? df_term(mu, exp2(ehi), kind) : 0.0);
        bool ok = (dlo > target) && (dhi < target);
        for (int it = 0; it < 80 && ok; it++) {
            double mid = 0.5 * (elo + ehi);
            double v = warp_sum(tid < d ? df_term(mu, exp2(mid), kind) : 0.0);
            if (v > target) elo = mid;
            else ehi = mid;
        }
        if (tid == 0) {
            if (!ok) { fail = 1; cwb_dev_fail(status, CWB_ECALIB); }
            s_lambda = exp2(0.5 * (elo + ehi));
        }
    }
    __syncthreads();
    if (fail) return;
    // Newton polish of the DRO root on the definition df(lambda) = tr(A^-1 G)
    // (supp. P:L316): the whitened eigenvalues carry cond(G + D) * eps error,
    // the dense trace only cond(A) * eps.  Two steps, then the cached inverse.
    __shared__ double red[32];
    for (int it = 0; it <= 2; it++) {
        const double lam = s_lambda;
        // A = G + lambda D -> Cholesky -> A^{-1} = L^{-T} L^{-1}  (cached)
        for (int e = tid; e < d * d; e += nthr) { const int a = e / d, b = e % d; P[a][b] = G[a][b] + lam * Dm[a][b]; }
        __syncthreads();
        blk_cholesky(P, d, &fail);
        if (fail) { if (tid == 0) cwb_dev_fail(status, CWB_ECALIB); return; }
        blk_tri_inverse(P, W, d);
        for (int e = tid; e < d * d; e += nthr) {  // P <- A^{-1} (symmetric)
            const int i = e / d, c = e % d;
            if (c <= i) {
                double s = 0.0;
                for (int q = i; q < d; q++) s += W[q][i] * W[q][c];
                P[i][c] = s;
                P[c][i] = s;
            }
        }
        __syncthreads();
        if (it == 2) {
            for (int e = tid; e < d * d; e += nthr) Ainv_out[(size_t)k * d * d + e] = P[e / d][e % d];
            if (tid == 0) lambda_out[k] = lam;
            break;
        }
        for (int e = tid; e < d * d; e += nthr) {  // M <- X = A^-1 G,  W <- A^-1 D
            const int i = e / d, c = e % d;
            double x = 0.0, y = 0.0;
            for (int q = 0; q < d; q++) { x += P[i][q] * G[q][c]; y += P[i][q] * Dm[q][c]; }
            M[i][c] = x;
            W[i][c] = y;
        }
        __syncthreads();
        // f = df - target, f' = d df / d lambda  (dX/dlambda = -A^-1 D X)
        double tX = 0.0, tXX = 0.0, tYX = 0.0, tXYX = 0.0;
        for (int e = tid; e < d * d; e += nthr) {
            const int i = e / d, c = e % d;
            if (i == c) tX += M[i][i];
            tXX += M[i][c] * M[c][i];
            double yx = 0.0, xy = 0.0;
            for (int q = 0; q < d; q++) { yx += W[i][q] * M[q][c]; xy += M[i][q] * W[q][c]; }
            if (i == c) tYX += yx;
            tXYX += xy * M[c][i];
        }
        double vals[4] = {tX, tXX, tYX, tXYX};
        double tot[4];
        for (int q = 0; q < 4; q++) {
            double v = warp_sum(vals[q]);
            if ((tid & 31) == 0) red[tid >> 5] = v;
            __syncthreads();
            double t = 0.0;
            for (int w = 0; w < (nthr >> 5); w++) t += red[w];
            tot[q] = t;
            __syncthreads();
        }
        double f, fp;
        if (kind == 2) { f = 2.0 * tot[0] - tot[1] - target; fp = -2.0 * tot[2] + 2.0 * tot[3]; }
        else { f = tot[0] - target; fp = -tot[2]; }
        if (tid == 0) {
            double nl = lam - f / fp;
            if (isfinite(nl) && nl > 0.5 * lam && nl < 2.0 * lam) s_lambda = nl;
        }
        __syncthreads();
    }
}

}  // namespace

// ===================================================================== host

static int smem_csr_warps(int ns, int max_warps) {
    // per-warp bin counters + totals must fit in ~200 KB of shared memory
    long budget = 200 * 1024;
    int w = max_warps;
    while (w > 1 && (long)(w + 1) * ns * 4 > budget) w--;
    return w;
}

int cwb_launch_csr(cwb_ctx* ctx, const void* idx, int32_t idx_bytes, int64_t n, int32_t K,
                   int32_t ns, uint32_t* cnt, int32_t* off, void* perm, int32_t perm_bytes,
                   cudaStream_t s) {
    const int threads = 1024;
    int nw = smem_csr_warps(ns, threads / 32);
    size_t smem = (size_t)(nw + 1) * ns * sizeof(uint32_t);
    if ((long)(nw + 1) * ns * 4 > 200 * 1024)
        return cwb_set_error(ctx, CWB_EUNSUPPORTED, "n* too large for the bin inversion kernel");
    const int* st = ctx ? ctx->d_status : nullptr;
#define CSR_CASE(IT, PT)                                                                         \
    {                                                                                            \
        auto kern = k_csr<IT, PT>;                                                               \
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);      \
        kern<<<K, threads, smem, s>>>((const IT*)idx, n, ns, nw, cnt, off, (PT*)perm, st);       \
    }
    if (idx_bytes == 1 && perm_bytes == 2) CSR_CASE(uint8_t, uint16_t)
    else if (idx_bytes == 1 && perm_bytes == 4) CSR_CASE(uint8_t, uint32_t)
    else if (idx_bytes == 2 && perm_bytes == 2) CSR_CASE(uint16_t, uint16_t)
    else CSR_CASE(uint16_t, uint32_t)
#undef CSR_CASE
    if (ctx) ctx->launches++;
    return cwb_check_launch(ctx, "k_csr");
}

int cwb_launch_bin_only(cwb_ctx* ctx, int* st, const double* x, int64_t n, int32_t K, int32_t ns,
                        double* lo, double* hi, double* z, double* bnd, void* idx, int32_t idx_bytes,
                        cudaStream_t s) {
    k_minmax<<<K, 512, 0, s>>>(x, n, lo, hi, st);
    k_design<<<K, 256, 0, s>>>(lo, hi, ns, z, bnd, st);
    int gx = (int)((n + 255) / 256);
    if (gx > 1184) gx = 1184;
    dim3 grid(gx, K);
    size_t smem = sizeof(double) * (size_t)(ns > 1 ? ns - 1 : 1);
    const bool use_smem = smem <= 48 * 1024;
    if (!use_smem) smem = 0;
    if (idx_bytes == 1) {
        if (use_smem) k_bin<uint8_t, true><<<grid, 256, smem, s>>>(x, n, ns, bnd, (uint8_t*)idx, st);
        else k_bin<uint8_t, false><<<grid, 256, 0, s>>>(x, n, ns, bnd, (uint8_t*)idx, st);
    } else {
        if (use_smem) k_bin<uint16_t, true><<<grid, 256, smem, s>>>(x, n, ns, bnd, (uint16_t*)idx, st);
        else k_bin<uint16_t, false><<<grid, 256, 0, s>>>(x, n, ns, bnd, (uint16_t*)idx, st);
    }
    if (ctx) ctx->launches += 3;
    return cwb_check_launch(ctx, "binning kernels");
}

int cwb_launch_init(cwb_ctx* c, const double* X, cudaStream_t s) {
    const int K = c->K, ns = c->n_star, d = c->d;
    int rc = cwb_launch_bin_only(c, c->d_status, X, c->n, K, ns, c->lo, c->hi, c->z, c->bnd, c->idx,
                                 c->idx_bytes, s);
    if (rc) return rc;
    rc = cwb_launch_csr(c, c->idx, c->idx_bytes, c->n, K, ns, c->cnt, c->off, c->perm,
                        c->perm_bytes, s);
    if (rc) return rc;
    k_basis<<<K, 128, sizeof(int32_t) * ns, s>>>(c->z, c->lo, c->hi, ns, c->degree, c->n_knots, d,
                                                 c->Zb, c->zj0, c->Zs, c->lwin, c->d_status);
    k_gram<<<K, 256, 0, s>>>(c->Zb, c->cnt, ns, d, c->lwin, c->G, c->d_status);
    k_dro<<<K, 256, 0, s>>>(c->G, d, c->df, c->df_kind, c->lambda, c->Ainv, c->eig, c->d_status);
    c->launches += 3;
    return cwb_check_launch(c, "pool kernels");
}
