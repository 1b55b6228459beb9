// cwb_init.cu -- one-off pool construction on the device (I1-I7).
//
//   I1 k_minmax_part / _fin   per-learner min / max of x (HBM-bound, all SMs)
//   I1b k_distinct  n*_k = min(n*, #distinct values)                S:L143 (reading N1)
//   I2 k_design   design points z and bin boundaries
//   I3 k_bin      index vector (nearest design point, then exact boundary comparisons)
//   I4 k_csr      bin inversion: rows of every bin, ascending      (binning as a hash map)
//   I5 k_basis    cubic B-spline basis at the design points
//   I6 k_gram     G = Zb^T diag(cnt) Zb  (binMatMat, w = 1)
//   I7 k_lambda   df(lambda) = df by Newton on the definition, (G + lambda D)^-1   supp. P:L314-319
//
// Everything here runs once per data set and is shared by all B
// replications.  Bit-exactness with the paper's fp64 definitions matters for
// I2/I3 (integer bin decisions): they use explicit round-to-nearest
// intrinsics so that no FMA contraction changes a rounding.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "cwb_internal.cuh"

namespace {

// ---------------------------------------------------------------- I1 min/max
// HBM-bound: blocks of every learner reduce contiguous row ranges (4 loads in flight per
// thread), k_minmax_fin combines the partials and records ENONFINITE / EDEGENERATE.
constexpr int kMMT = 256;

__global__ void __launch_bounds__(kMMT) k_minmax_part(const double* __restrict__ X, int64_t n, int nb,
                                                      double* __restrict__ part) {
    const int k = blockIdx.y, b = blockIdx.x;
    const double* x = X + (size_t)k * n;
    const int64_t per = (n + nb - 1) / nb, r0 = min(n, (int64_t)b * per), r1 = min(n, r0 + per);
    double mn = INFINITY, mx = -INFINITY;
    bool bad = false;
    int64_t i = r0 + threadIdx.x;
    for (; i + 3 * kMMT < r1; i += 4 * kMMT) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; u++) v[u] = __ldcs(x + i + u * kMMT);
#pragma unroll
        for (int u = 0; u < 4; u++) {
            bad |= !isfinite(v[u]);
            mn = fmin(mn, v[u]);
            mx = fmax(mx, v[u]);
        }
    }
    for (; i < r1; i += kMMT) {
        const double v = __ldcs(x + i);
        bad |= !isfinite(v);
        mn = fmin(mn, v);
        mx = fmax(mx, v);
    }
    __shared__ double smn[kMMT / 32], smx[kMMT / 32];
    __shared__ int sbad;
    if (threadIdx.x == 0) sbad = 0;
    __syncthreads();
    if (bad) sbad = 1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { smn[w] = mn; smx[w] = mx; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < kMMT / 32; q++) { mn = fmin(mn, smn[q]); mx = fmax(mx, smx[q]); }
        double* o = part + ((size_t)k * nb + b) * 3;
        o[0] = mn;
        o[1] = mx;
        o[2] = sbad ? 1.0 : 0.0;
    }
}

__global__ void k_minmax_fin(const double* __restrict__ part, int nb, double* lo, double* hi, int* status) {
    const int k = blockIdx.x, lane = threadIdx.x;
    double mn = INFINITY, mx = -INFINITY, bad = 0.0;
    for (int b = lane; b < nb; b += 32) {
        const double* q = part + ((size_t)k * nb + b) * 3;
        mn = fmin(mn, q[0]);
        mx = fmax(mx, q[1]);
        bad = fmax(bad, q[2]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        bad = fmax(bad, __shfl_xor_sync(0xffffffffu, bad, o));
    }
    if (lane == 0) {
        lo[k] = mn;
        hi[k] = mx;
        if (bad != 0.0) cwb_dev_fail(status, CWB_ENONFINITE);
        else if (!(mn < mx)) cwb_dev_fail(status, CWB_EDEGENERATE);
    }
}

// z_l = lo + (l/(n*-1)) (hi - lo), z_{n*-1} = hi, each operation rounded once
__device__ __forceinline__ double design_point(double lo, double hi, int l, int ns) {
    if (l == ns - 1) return hi;
    double t = __ddiv_rn((double)l, (double)(ns - 1));
    return __dadd_rn(lo, __dmul_rn(t, __dsub_rn(hi, lo)));
}

// ------------------------------------------- I1b distinct values (n* clamp)
// S:L143 (reading N1): the bins of learner k are those of
// n*_k = min(n*, #distinct values of x_k).  One CTA per learner inserts the values
// into an open-addressing hash set of H = 2^m >= 2 (n* + T) slots (shared memory, or
// the global scratch `gtab` when it does not fit) and stops as soon as n* distinct
// values are seen -- a continuous feature exits after its first few thousand rows.
// The T threads see the stop flag at their next row, so at most n* + T - 1 keys are
// ever inserted: the load factor stays <= 1/2 and every probe sequence ends.
// Keys are the value bits with -0.0 folded into +0.0; empty = all ones (a NaN: the
// values are finite, k_minmax has checked).  The count is exact below n*.
constexpr unsigned long long kEmptyKey = ~0ull;

__global__ void k_distinct(const double* __restrict__ X, int64_t n, int ns, int hbits,
                           unsigned long long* __restrict__ gtab, int32_t* __restrict__ nsk, const int* status) {
    extern __shared__ unsigned long long htab_s[];
    __shared__ int s_count;
    __shared__ volatile int s_full;
    if (status && *status) return;
    const int k = blockIdx.x;
    const uint32_t H = 1u << hbits, mask = H - 1u;
    unsigned long long* tab = gtab ? gtab + (size_t)k * H : htab_s;
    for (uint32_t e = threadIdx.x; e < H; e += blockDim.x) tab[e] = kEmptyKey;
    if (threadIdx.x == 0) { s_count = 0; s_full = 0; }
    __syncthreads();
    const double* x = X + (size_t)k * n;
    for (int64_t i = threadIdx.x; i < n && !s_full; i += blockDim.x) {
        const double v = x[i];
        const unsigned long long key = (unsigned long long)__double_as_longlong(v == 0.0 ? 0.0 : v);
        uint32_t h = (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> (64 - hbits));
        for (uint32_t probe = 0;; probe++) {
            if (probe >= H) {  // unreachable at load <= 1/2; never spin
                cwb_dev_fail(const_cast<int*>(status), CWB_ECUDA);
                s_full = 1;
                break;
            }
            unsigned long long cur = gtab ? __ldcg(tab + h) : tab[h];
            if (cur == key) break;
            if (cur == kEmptyKey) {
                cur = atomicCAS(tab + h, kEmptyKey, key);
                if (cur == kEmptyKey) {
                    if (atomicAdd(&s_count, 1) + 1 >= ns) s_full = 1;
                    break;
                }
                if (cur == key) break;
            }
            h = (h + 1u) & mask;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) nsk[k] = s_count < ns ? s_count : ns;
}

// ---------------------------------------------------------- I2 design points
// nsk (NULL: n* for every learner): the design points of n*_k = nsk[k]; the slots
// l >= n*_k are padding, z = hi and bnd = +inf (no row is binned there).
__global__ void k_design(const double* lo_, const double* hi_, int ns, const int32_t* nsk, double* z, double* bnd,
                         const int* status) {
    if (status && *status) return;
    const int k = blockIdx.x;
    const double lo = lo_[k], hi = hi_[k];
    const int nk = nsk ? nsk[k] : ns;
    for (int l = threadIdx.x; l < ns; l += blockDim.x) {
        double zl = l < nk ? design_point(lo, hi, l, nk) : hi;
        z[(size_t)k * ns + l] = zl;
        if (l < ns - 1) {
            double b = INFINITY;
            if (l < nk - 1) {
                double zr = design_point(lo, hi, l + 1, nk);
                b = __dadd_rn(zl, __ddiv_rn(__dsub_rn(zr, zl), 2.0));
            }
            bnd[(size_t)k * (ns - 1) + l] = b;
        }
    }
}

// ------------------------------------------------------------ I3 index vector
// idx(x) = smallest l with x <= bnd_l, else n*-1 (P:L861 closed-right bins).  The search
// starts at the nearest design point by arithmetic, g = round((x - lo) (n*_k - 1) / (hi - lo)),
// and walks to the exact answer by comparisons with bnd (non-decreasing): down while
// x <= bnd_{g-1}, up while x > bnd_g -- the same index as a binary search over bnd, in one or
// two shared-memory loads instead of log2 n*.  Padding boundaries (l >= n*_k - 1) are +inf.
template <typename IdxT, bool SMEM>
__global__ void k_bin(const double* __restrict__ X, int64_t n, int ns, const double* __restrict__ bnd,
                      const double* __restrict__ lo_, const double* __restrict__ hi_,
                      const int32_t* __restrict__ nsk, IdxT* __restrict__ idx, const int* status) {
    extern __shared__ double sb[];
    if (status && *status) return;
    const int k = blockIdx.y;
    const double* bk = bnd + (size_t)k * (ns - 1);
    if (SMEM) {
        for (int l = threadIdx.x; l < ns - 1; l += blockDim.x) sb[l] = bk[l];
        __syncthreads();
    }
    const double* bs = SMEM ? sb : bk;
    const int nk = nsk ? nsk[k] : ns;
    const double lo = lo_[k], scale = (double)(nk - 1) / (hi_[k] - lo);
    const double* x = X + (size_t)k * n;
    IdxT* out = idx + (size_t)k * n;
    const int64_t per = (n + gridDim.x - 1) / gridDim.x, r0 = min(n, (int64_t)blockIdx.x * per),
                  r1 = min(n, r0 + per);
    auto bin = [&](double v) {
        const double t = (v - lo) * scale + 0.5;
        int g = t >= 0.0 ? (t < (double)(nk - 1) ? (int)t : nk - 1) : 0;
        while (g > 0 && v <= bs[g - 1]) g--;
        while (g < ns - 1 && v > bs[g]) g++;
        return (IdxT)g;
    };
    const int T = blockDim.x;
    int64_t i = r0 + threadIdx.x;
    for (; i + 3 * T < r1; i += 4 * T) {  // four loads in flight per thread
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; u++) v[u] = __ldcs(x + i + u * T);
#pragma unroll
        for (int u = 0; u < 4; u++) out[i + u * T] = bin(v[u]);
    }
    for (; i < r1; i += T) out[i] = bin(__ldcs(x + i));
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
                        const int32_t* __restrict__ nsk, int deg, int nk, int d, double* Zb, int32_t* zj0,
                        double* Zs, int32_t* lwin, const int* status) {
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
        // first non-zero basis (w0 is clamped to d - 4 for degree < 3); padding design points
        // (l >= n*_k) are in no basis window
        sj0[l] = (nsk && l >= nsk[k]) ? (1 << 30) : (j0 < 0 ? 0 : j0);
    }
    __syncthreads();
    // design-point window of basis j: l with j - deg <= j0(l) <= j (j0 non-decreasing), i.e. the
    // deg + 1 knot intervals of its support
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
        int a = 0, b = ns;  // first l with j0[l] >= j - deg
        while (a < b) { int m = (a + b) >> 1; if (sj0[m] >= j - deg) b = m; else a = m + 1; }
        int lb = a;
        a = lb; b = ns;     // first l with j0[l] > j
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

// ------------------------------------------- I7 df -> lambda, cached inverse
// One warp per learner (no block barriers).  df(lambda) is evaluated by its
// definition (supp.): A = G + lambda D, df1 = tr(A^-1 G),
// df2 = tr(2 A^-1 G - (A^-1 G)^2), with its exact derivative
// d tr(A^-1 G)/d lambda = -tr(A^-1 D A^-1 G).  The root of df(lambda) = df
// ("must be solved numerically") is found by safeguarded Newton
// in t = log(lambda).  The paper's Demmler-Reinsch route makes each
// df evaluation O(d) after an O(d^3) eigen-decomposition, a CPU trade-off; a
// warp evaluates the O(d^3) definition in a few microseconds and Newton needs
// a handful of steps, so the eigen-decomposition is not used.
// The inverse of the final A is cached for the iterations.
#define DS 33  // padded shared row stride

__device__ __forceinline__ double dpen(int a, int b, int d) {
    // D = Delta^T Delta, Delta rows (.., 1, -2, 1, ..)  (supp. P:L312)
    double v = 0.0;
    for (int i = max(0, max(a, b) - 2); i <= min(a, b) && i + 2 < d; i++) {
        const double ca = (a == i) ? 1.0 : (a == i + 1) ? -2.0 : 1.0;
        const double cb = (b == i) ? 1.0 : (b == i + 1) ? -2.0 : 1.0;
        v += ca * cb;
    }
    return v;
}

struct LamEval { double f, fp; bool ok; };

#define BW 3  // half-bandwidth of G (cubic B-splines overlap 4 design windows) and of D (2)

// Banded Cholesky of A = G + lambda D (lane 0), then lane c solves A x = b_c
// for the columns of G (-> X = A^-1 G) and of D (-> Y = A^-1 D).
// f(t) = df(e^t) - target, f'(t) = lambda d df / d lambda,
// d tr(X)/d lambda = -tr(Y X), d tr(X^2)/d lambda = -2 tr(X Y X).
// The factor keeps the last three rows in registers (no shared-memory round trip
// in the dependency chain) and uses rsqrt for the pivots (no division).
// Lb[j*4 + q] = L[j][j-q] (q = 0..3), inv[j] = 1 / L[j][j]; Lb is zero beyond row d.
__device__ void band_factor(double lam, int d, double (*Gs)[DS], double (*Dm)[DS], double* Lb, double* inv,
                            bool* ok_out) {
    if ((threadIdx.x & 31) == 0) {
        bool ok = true;
        double r1_1 = 0.0, r1_2 = 0.0, r2_1 = 0.0;  // L[j-1][j-2], L[j-1][j-3], L[j-2][j-3]
        double i1 = 0.0, i2 = 0.0, i3 = 0.0;        // inverse pivots of rows j-1, j-2, j-3
        for (int j = 0; j < d; j++) {
            const double a0 = Gs[j][j] + lam * Dm[j][j];
            const double a1 = j >= 1 ? Gs[j][j - 1] + lam * Dm[j][j - 1] : 0.0;
            const double a2 = j >= 2 ? Gs[j][j - 2] + lam * Dm[j][j - 2] : 0.0;
            const double a3 = j >= 3 ? Gs[j][j - 3] + lam * Dm[j][j - 3] : 0.0;
            const double x3 = a3 * i3;
            const double x2 = (a2 - x3 * r2_1) * i2;
            const double x1 = (a1 - x3 * r1_2 - x2 * r1_1) * i1;
            const double v = a0 - x3 * x3 - x2 * x2 - x1 * x1;
            ok &= v > 0.0;
            const double vi = rsqrt(fmax(v, 1e-300));
            Lb[j * 4 + 0] = v * vi;
            Lb[j * 4 + 1] = x1;
            Lb[j * 4 + 2] = x2;
            Lb[j * 4 + 3] = x3;
            inv[j] = vi;
            r2_1 = r1_1;  // row j-1 becomes row j-2: its L[.][.-1]
            r1_1 = x1;
            r1_2 = x2;
            i3 = i2; i2 = i1; i1 = vi;
        }
        *ok_out = ok;
    }
    __syncwarp();
}

// x = A^-1 b for b = column c of B (read through the functor), result in column c of Xs
template <typename Fb>
__device__ __forceinline__ void band_solve(int d, const double* Lb, const double* inv, Fb b, double (*Xs)[DS], int c) {
    double z1 = 0.0, z2 = 0.0, z3 = 0.0;
    for (int j = 0; j < d; j++) {  // L z = b
        const double v = b(j) - Lb[j * 4 + 1] * z1 - Lb[j * 4 + 2] * z2 - Lb[j * 4 + 3] * z3;
        const double z = v * inv[j];
        Xs[j][c] = z;
        z3 = z2; z2 = z1; z1 = z;
    }
    double x1 = 0.0, x2 = 0.0, x3 = 0.0;
    for (int j = d - 1; j >= 0; j--) {  // L^T x = z (Lb rows beyond d are zero)
        const double v = Xs[j][c] - Lb[(j + 1) * 4 + 1] * x1 - Lb[(j + 2) * 4 + 2] * x2 - Lb[(j + 3) * 4 + 3] * x3;
        const double x = v * inv[j];
        Xs[j][c] = x;
        x3 = x2; x2 = x1; x1 = x;
    }
}

__device__ LamEval lam_eval(double t, int d, double target, int kind, double (*Gs)[DS], double (*Dm)[DS],
                            double (*Xs)[DS], double (*Ys)[DS], double* Lb, double* inv) {
    const int i = threadIdx.x & 31;
    const double lam = exp(t);
    __shared__ bool s_ok;
    band_factor(lam, d, Gs, Dm, Lb, inv, &s_ok);
    if (i < d) {
        band_solve(d, Lb, inv, [&](int j) { return Gs[j][i]; }, Xs, i);
        band_solve(d, Lb, inv, [&](int j) { return Dm[j][i]; }, Ys, i);
    }
    __syncwarp();
    double tX = 0.0, tYX = 0.0, tXX = 0.0, tXYX = 0.0;
    if (i < d) {
        tX = Xs[i][i];
        for (int j = 0; j < d; j++) {
            tYX += Ys[i][j] * Xs[j][i];
            if (kind == 2) {
                tXX += Xs[i][j] * Xs[j][i];
                double xy = 0.0;
                for (int q = 0; q < d; q++) xy += Xs[i][q] * Ys[q][j];
                tXYX += xy * Xs[j][i];
            }
        }
    }
    tX = warp_sum(tX);
    tYX = warp_sum(tYX);
    tXX = warp_sum(tXX);
    tXYX = warp_sum(tXYX);
    __syncwarp();
    LamEval e;
    e.ok = s_ok;
    if (kind == 2) { e.f = 2.0 * tX - tXX - target; e.fp = lam * (-2.0 * tYX + 2.0 * tXYX); }
    else { e.f = tX - target; e.fp = -lam * tYX; }
    return e;
}

__global__ void k_lambda(const double* __restrict__ Gall, int d, double target, int kind,
                         double* lambda_out, double* Ainv_out, double* Cb_out, int* status) {
    __shared__ double Gs[CWB_MAX_D][DS], Dm[CWB_MAX_D][DS], Xs[CWB_MAX_D][DS], Ys[CWB_MAX_D][DS];
    __shared__ double Lb[(CWB_MAX_D + 4) * 4], inv[CWB_MAX_D];
    if (status && *status) return;
    const int k = blockIdx.x, i = threadIdx.x;
    for (int e = i; e < (CWB_MAX_D + 4) * 4; e += 32) Lb[e] = 0.0;  // zero band beyond row d
    if (i < d)
        for (int c = 0; c < d; c++) {
            Gs[i][c] = Gall[((size_t)k * d + i) * d + c];
            Dm[i][c] = dpen(i, c, d);
        }
    __syncwarp();
    const double trG = warp_sum(i < d ? Gs[i][i] : 0.0);
    const double trD = warp_sum(i < d ? Dm[i][i] : 0.0);
    const double t0 = log(fmax(trG, 1e-300) / fmax(trD, 1e-300));
    double t = t0;
    double tlo = -INFINITY, thi = INFINITY;  // f(tlo) > 0 > f(thi)
    bool done = false, fail = false;
    int it = 0;
    for (; it < 80 && !done; it++) {
        LamEval e = lam_eval(t, d, target, kind, Gs, Dm, Xs, Ys, Lb, inv);
#ifdef CWB_DEBUG_LAMBDA
        if (i == 0) printf("k=%d it=%d t=%.17g f=%.3e fp=%.3e ok=%d\n", k, it, t, e.f, e.fp, (int)e.ok);
#endif
        if (!e.ok || !isfinite(e.f)) {
            // A not numerically SPD: above the start the penalty dominates (lambda too high, its
            // null space meets G's small directions), below it G's rank deficiency does (too low)
            if (t > t0) { thi = t; t = isfinite(tlo) ? 0.5 * (t + tlo) : t - 4.0; }
            else { tlo = t; t = isfinite(thi) ? 0.5 * (t + thi) : t + 4.0; }
            if (t > 120.0 || t < -120.0) { fail = true; break; }
            continue;
        }
        if (fabs(e.f) <= 1e-13 * target) { done = true; break; }
        if (e.f > 0.0) tlo = t; else thi = t;
        double tn = t - e.f / e.fp;
        if (!isfinite(tn)) tn = e.f > 0.0 ? t + 4.0 : t - 4.0;
        tn = fmin(fmax(tn, t - 6.0), t + 6.0);  // at most a factor e^6 in lambda per step (flat df when G is rank-deficient)
        const bool inside = tn > tlo && tn < thi;
        if (!inside) {
            if (isfinite(tlo) && isfinite(thi)) tn = 0.5 * (tlo + thi);
            else tn = (e.f > 0.0) ? t + 4.0 : t - 4.0;
        }
        if (fabs(tn - t) <= 1e-15 * fmax(1.0, fabs(t))) {  // step below resolution: stop at tn
            t = tn;
            e = lam_eval(t, d, target, kind, Gs, Dm, Xs, Ys, Lb, inv);
            done = e.ok;
            fail = !e.ok || fabs(e.f) > 1e-9;
            break;
        }
        if (tn < -120.0 || tn > 120.0) { fail = true; break; }
        t = tn;
    }
    if (!done || fail) {
        if (i == 0) cwb_dev_fail(status, CWB_ECALIB);
        return;
    }
    // cached inverse: columns of A^-1 by banded solves, symmetrised
    if (i < d) band_solve(d, Lb, inv, [&](int j) { return j == i ? 1.0 : 0.0; }, Xs, i);
    __syncwarp();
    const double lam = exp(t);
    if (i == 0) lambda_out[k] = lam;
    if (i < d)
        for (int c = 0; c < d; c++)
            Ainv_out[((size_t)k * d + i) * d + c] = 0.5 * (Xs[i][c] + Xs[c][i]);
    // Selection factor: C C^T = G + 2 lambda D (banded Cholesky), so that for theta = A^-1 s
    // 2 theta^T s - theta^T G theta = theta^T (2A - G) theta = |C^T theta|^2.
    __shared__ bool s_ok2;
    band_factor(2.0 * lam, d, Gs, Dm, Lb, inv, &s_ok2);
    if (!s_ok2) {
        if (i == 0) cwb_dev_fail(status, CWB_ECALIB);
        return;
    }
    if (i < d)
        for (int q = 0; q < 4; q++)  // Cb[j][q] = C[j+q][j] (Lb[row*4 + q] = C[row][row-q])
            Cb_out[((size_t)k * d + i) * 4 + q] = (q <= BW && i + q < d) ? Lb[(i + q) * 4 + q] : 0.0;
}

// Windows of the basis functions: ZT[k][w][j] = Zb[k][lb_j + w][j] for the design points
// lb_j <= l < le_j where B_j(z_l) can be non-zero (lwin), zero-padded to W.
__global__ void k_zt(const double* __restrict__ Zb, const int32_t* __restrict__ lwin, int ns, int d, int W,
                     double* __restrict__ ZT, int* status) {
    if (status && *status) return;
    const int k = blockIdx.x;
    for (int e = threadIdx.x; e < W * d; e += blockDim.x) {
        const int w = e / d, j = e - w * d;
        const int lb = lwin[((size_t)k * d + j) * 2], le = lwin[((size_t)k * d + j) * 2 + 1];
        if (w == 0 && le - lb > W) cwb_dev_fail(status, CWB_EUNSUPPORTED);
        ZT[((size_t)k * W + w) * d + j] = (lb + w < le) ? Zb[((size_t)k * ns + lb + w) * d + j] : 0.0;
    }
}

// Training-row statistics for HCWB (Alg. 3): counts of the rows with mask == 0 per bin
// (binMatMat with 0/1 observation weights).  Integer atomics: exact.
template <typename IdxT>
__global__ void k_count_masked(const IdxT* __restrict__ idx, const uint8_t* __restrict__ mask, int64_t n, int ns,
                               uint32_t* __restrict__ cnt, const int* status) {
    extern __shared__ uint32_t hc[];
    if (status && *status) return;
    const int k = blockIdx.y;
    for (int l = threadIdx.x; l < ns; l += blockDim.x) hc[l] = 0u;
    __syncthreads();
    const IdxT* ik = idx + (size_t)k * n;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (!mask[i]) atomicAdd(&hc[ik[i]], 1u);
    __syncthreads();
    for (int l = threadIdx.x; l < ns; l += blockDim.x)
        if (hc[l]) atomicAdd(&cnt[(size_t)k * ns + l], hc[l]);
}

// (G + lambda D)^-1 for a given lambda (one warp per learner): the cached inverse of the
// training-row learners, with the lambda calibrated on all rows (HCWB readings)
// (Cb_out != NULL: also the band of C, C C^T = G + 2 lambda D, as k_lambda's selection factor)
__global__ void k_inverse_fixed(const double* __restrict__ Gall, const double* __restrict__ lambda, int d,
                                double* __restrict__ Ainv_out, int* status, double* __restrict__ Cb_out = nullptr) {
    __shared__ double Gs[CWB_MAX_D][DS], Dm[CWB_MAX_D][DS], Xs[CWB_MAX_D][DS];
    __shared__ double Lb[(CWB_MAX_D + 4) * 4], inv[CWB_MAX_D];
    __shared__ bool s_ok;
    if (status && *status) return;
    const int k = blockIdx.x, i = threadIdx.x;
    for (int e = i; e < (CWB_MAX_D + 4) * 4; e += 32) Lb[e] = 0.0;
    if (i < d)
        for (int c = 0; c < d; c++) {
            Gs[i][c] = Gall[((size_t)k * d + i) * d + c];
            Dm[i][c] = dpen(i, c, d);
        }
    __syncwarp();
    band_factor(lambda[k], d, Gs, Dm, Lb, inv, &s_ok);
    if (!s_ok) {
        if (i == 0) cwb_dev_fail(status, CWB_ECALIB);
        return;
    }
    if (i < d) band_solve(d, Lb, inv, [&](int j) { return j == i ? 1.0 : 0.0; }, Xs, i);
    __syncwarp();
    if (i < d)
        for (int c = 0; c < d; c++) Ainv_out[((size_t)k * d + i) * d + c] = 0.5 * (Xs[i][c] + Xs[c][i]);
    if (!Cb_out) return;
    __syncwarp();
    __shared__ bool s_ok2;
    band_factor(2.0 * lambda[k], d, Gs, Dm, Lb, inv, &s_ok2);
    if (!s_ok2) {
        if (i == 0) cwb_dev_fail(status, CWB_ECALIB);
        return;
    }
    if (i < d)
        for (int q = 0; q < 4; q++)  // Cb[j][q] = C[j+q][j]
            Cb_out[((size_t)k * d + i) * 4 + q] = (q <= BW && i + q < d) ? Lb[(i + q) * 4 + q] : 0.0;
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

namespace {
// ------------------------------------------- I4 bin inversion, chunked (large n)
// The same stable counting sort as k_csr spread over (chunk, learner) CTAs: chunk c of
// learner k holds rows [c C, (c+1) C).  k_csrc_count: per-chunk bin counts; k_csrc_scan:
// per learner the bin totals, the offsets off[l] and the first slot of every (chunk, bin),
// off[l] + rows of bin l in the chunks before; k_csrc_scatter: the chunk's rows sorted by
// bin in shared memory (per-warp histograms + __match_any_sync ranks: stable), then
// written out run by run (consecutive threads, consecutive slots).  The output is
// bit-identical to k_csr's (a stable sort is unique).
constexpr int kCsrC = 16384;  // rows per chunk
constexpr int kCsrT = 512;

template <typename IdxT>
__global__ void __launch_bounds__(kCsrT) k_csrc_count(const IdxT* __restrict__ idx, int64_t n, int ns, int nch,
                                                      uint32_t* __restrict__ ccnt, const int* status) {
    extern __shared__ uint32_t hc2[];
    if (status && *status) return;
    const int c = blockIdx.x, k = blockIdx.y;
    for (int l = threadIdx.x; l < ns; l += kCsrT) hc2[l] = 0;
    __syncthreads();
    const IdxT* id = idx + (size_t)k * n;
    const int64_t r0 = (int64_t)c * kCsrC, r1 = min(n, r0 + kCsrC);
    for (int64_t i = r0 + threadIdx.x; i < r1; i += kCsrT) atomicAdd(&hc2[id[i]], 1u);
    __syncthreads();
    uint32_t* o = ccnt + ((size_t)k * nch + c) * ns;
    for (int l = threadIdx.x; l < ns; l += kCsrT) o[l] = hc2[l];
}

__global__ void __launch_bounds__(1024) k_csrc_scan(uint32_t* __restrict__ ccnt, int64_t n, int ns, int nch,
                                                    uint32_t* __restrict__ cnt_out, int32_t* __restrict__ off_out,
                                                    const int* status) {
    extern __shared__ uint32_t tot2[];
    __shared__ uint32_t wsum[32];
    if (status && *status) return;
    const int k = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5, nthr = blockDim.x;
    uint32_t* cc = ccnt + (size_t)k * nch * ns;
    for (int l = threadIdx.x; l < ns; l += nthr) {  // chunk-exclusive prefix per bin, totals
        uint32_t run = 0;
        for (int c = 0; c < nch; c++) {
            const uint32_t v = cc[(size_t)c * ns + l];
            cc[(size_t)c * ns + l] = run;
            run += v;
        }
        tot2[l] = run;
        cnt_out[(size_t)k * ns + l] = run;
    }
    __syncthreads();
    const int per = (ns + nthr - 1) / nthr;  // exclusive scan of the totals: off[l]
    const int b0 = threadIdx.x * per, b1 = min(ns, b0 + per);
    uint32_t local = 0;
    for (int b = b0; b < b1; b++) local += tot2[b];
    uint32_t inc = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    if (w == 0) {
        const uint32_t v = lane < (nthr >> 5) ? wsum[lane] : 0u;
        uint32_t sc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, sc, o);
            if (lane >= o) sc += t;
        }
        wsum[lane] = sc - v;
    }
    __syncthreads();
    uint32_t base = wsum[w] + inc - local;
    int32_t* off = off_out + (size_t)k * (ns + 1);
    for (int b = b0; b < b1; b++) {
        const uint32_t c = tot2[b];
        tot2[b] = base;
        off[b] = (int32_t)base;
        base += c;
    }
    if (threadIdx.x == 0) off[ns] = (int32_t)n;
    __syncthreads();
    for (int l = threadIdx.x; l < ns; l += nthr)
        for (int c = 0; c < nch; c++) cc[(size_t)c * ns + l] += tot2[l];
}

// shared memory: hist [nw][ns], lofs [ns], gst [ns], srow [C] (PermT), sbin [C] (u16)
template <typename IdxT, typename PermT>
__global__ void __launch_bounds__(kCsrT) k_csrc_scatter(const IdxT* __restrict__ idx, int64_t n, int ns, int nch,
                                                        int nw_use, const uint32_t* __restrict__ cst,
                                                        PermT* __restrict__ perm_out, const int* status) {
    extern __shared__ uint32_t sm2[];
    __shared__ uint32_t wsum[32];
    if (status && *status) return;
    const int c = blockIdx.x, k = blockIdx.y, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t* hist = sm2;
    uint32_t* lofs = hist + (size_t)nw_use * ns;
    uint32_t* gst = lofs + ns;
    PermT* srow = reinterpret_cast<PermT*>(gst + ns);
    uint16_t* sbin = reinterpret_cast<uint16_t*>(srow + kCsrC);
    const IdxT* id = idx + (size_t)k * n;
    const int64_t r0 = (int64_t)c * kCsrC, r1 = min(n, r0 + kCsrC);
    const int rows = (int)(r1 - r0);
    for (int a = threadIdx.x; a < nw_use * ns; a += kCsrT) hist[a] = 0;
    const uint32_t* cs = cst + ((size_t)k * nch + c) * ns;
    for (int l = threadIdx.x; l < ns; l += kCsrT) gst[l] = cs[l];
    __syncthreads();
    const int L = (rows + nw_use - 1) / nw_use;
    const int q0 = w * L, q1 = min(rows, q0 + L);
    if (w < nw_use)
        for (int q = q0 + lane; q < q1; q += 32) atomicAdd(&hist[(size_t)w * ns + id[r0 + q]], 1u);
    __syncthreads();
    // per bin: exclusive prefix over warps (hist -> warp base within the bin), bin totals in lofs
    for (int b = threadIdx.x; b < ns; b += kCsrT) {
        uint32_t run = 0;
        for (int q = 0; q < nw_use; q++) {
            const uint32_t v = hist[(size_t)q * ns + b];
            hist[(size_t)q * ns + b] = run;
            run += v;
        }
        lofs[b] = run;
    }
    __syncthreads();
    {   // exclusive scan of the bin totals: local offsets of the bins in the chunk's sorted order
        const int per = (ns + kCsrT - 1) / kCsrT;
        const int b0 = threadIdx.x * per, b1 = min(ns, b0 + per);
        uint32_t local = 0;
        for (int b = b0; b < b1; b++) local += lofs[b];
        uint32_t inc = local;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        if (lane == 31) wsum[w] = inc;
        __syncthreads();
        if (w == 0) {
            const uint32_t v = lane < kCsrT / 32 ? wsum[lane] : 0u;  // wsum has 32 slots
            uint32_t sc = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, sc, o);
                if (lane >= o) sc += t;
            }
            wsum[lane] = sc - v;
        }
        __syncthreads();
        uint32_t base = wsum[w] + inc - local;
        for (int b = b0; b < b1; b++) {
            const uint32_t t = lofs[b];
            lofs[b] = base;
            base += t;
        }
    }
    __syncthreads();
    for (int a = threadIdx.x; a < nw_use * ns; a += kCsrT) hist[a] += lofs[a % ns];
    __syncthreads();
    if (w < nw_use) {  // stable local slots: warps own contiguous row ranges, lanes ranked by match_any
        uint32_t* mybase = hist + (size_t)w * ns;
        for (int s0 = q0; s0 < q1; s0 += 32) {
            const int q = s0 + lane;
            const bool valid = q < q1;
            const uint32_t b = valid ? (uint32_t)id[r0 + q] : 0xffffffffu;
            const uint32_t mask = __match_any_sync(0xffffffffu, b);
            const uint32_t lt = mask & ((1u << lane) - 1u);
            if (valid) {
                const uint32_t slot = mybase[b] + __popc(lt);
                srow[slot] = (PermT)(r0 + q);
                sbin[slot] = (uint16_t)b;
            }
            __syncwarp();
            if (valid && lt == 0) mybase[b] += __popc(mask);
            __syncwarp();
        }
    }
    __syncthreads();
    PermT* perm = perm_out + (size_t)k * n;
    for (int t = threadIdx.x; t < rows; t += kCsrT) {
        const uint32_t b = sbin[t];
        perm[gst[b] + (uint32_t)t - lofs[b]] = srow[t];
    }
}
}  // namespace

int cwb_launch_csr(cwb_ctx* ctx, const void* idx, int32_t idx_bytes, int64_t n, int32_t K,
                   int32_t ns, uint32_t* cnt, int32_t* off, void* perm, int32_t perm_bytes,
                   cudaStream_t s) {
    const int* st0 = ctx ? ctx->d_status : nullptr;
    static const bool chunked_ok = [] {  // CWB_CSR_CHUNKED=0: always the one-CTA-per-learner k_csr
        const char* e = getenv("CWB_CSR_CHUNKED");
        return !(e && e[0] == '0');
    }();
    if (chunked_ok && n > 4 * (int64_t)kCsrC && ns <= 65535) {  // chunked: (chunk, learner) CTAs over all SMs
        const int nch = (int)((n + kCsrC - 1) / kCsrC);
        const size_t fixed = (size_t)kCsrC * (perm_bytes + 2) + 2 * sizeof(uint32_t) * ns;
        int nw = kCsrT / 32;
        while (nw > 1 && fixed + sizeof(uint32_t) * (size_t)nw * ns > 220 * 1024) nw >>= 1;
        const size_t ssm = fixed + sizeof(uint32_t) * (size_t)nw * ns;
        if (ssm <= 220 * 1024) {
            uint32_t* ccnt = nullptr;
            if (cwb_alloc((void**)&ccnt, sizeof(uint32_t) * (size_t)K * nch * ns, s) != cudaSuccess)
                return cwb_set_error(ctx, CWB_ENOMEM, "bin inversion scratch allocation failed");
            const dim3 g(nch, K);
            if (idx_bytes == 1)
                k_csrc_count<uint8_t><<<g, kCsrT, sizeof(uint32_t) * ns, s>>>((const uint8_t*)idx, n, ns, nch, ccnt, st0);
            else
                k_csrc_count<uint16_t><<<g, kCsrT, sizeof(uint32_t) * ns, s>>>((const uint16_t*)idx, n, ns, nch, ccnt, st0);
            k_csrc_scan<<<K, 1024, sizeof(uint32_t) * ns, s>>>(ccnt, n, ns, nch, cnt, off, st0);
#define CSRC_CASE(IT, PT)                                                                                  \
            {                                                                                              \
                auto kern = k_csrc_scatter<IT, PT>;                                                        \
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);         \
                kern<<<g, kCsrT, ssm, s>>>((const IT*)idx, n, ns, nch, nw, ccnt, (PT*)perm, st0);          \
            }
            if (idx_bytes == 1 && perm_bytes == 2) CSRC_CASE(uint8_t, uint16_t)
            else if (idx_bytes == 1) CSRC_CASE(uint8_t, uint32_t)
            else if (perm_bytes == 2) CSRC_CASE(uint16_t, uint16_t)
            else CSRC_CASE(uint16_t, uint32_t)
#undef CSRC_CASE
            cwb_release(ccnt, s);
            if (ctx) ctx->launches += 3;
            return cwb_check_launch(ctx, "chunked bin inversion");
        }
    }
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
                        cudaStream_t s, int32_t* nsk) {
    // I1: ~8 blocks of 256 threads per SM over all learners
    const int nsm = cwb_num_sms();
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>((n + 4 * kMMT - 1) / (4 * kMMT),
                                                              (8LL * nsm + K - 1) / K));
    double* mmp = nullptr;
    if (cwb_alloc((void**)&mmp, sizeof(double) * 3 * (size_t)nb * K, s) != cudaSuccess)
        return cwb_set_error(ctx, CWB_ENOMEM, "min/max scratch allocation failed");
    k_minmax_part<<<dim3(nb, K), kMMT, 0, s>>>(x, n, nb, mmp);
    k_minmax_fin<<<K, 32, 0, s>>>(mmp, nb, lo, hi, st);
    cwb_release(mmp, s);
    unsigned long long* gtab = nullptr;
    if (nsk) {  // per-learner n* clamp
        const int T = 1024;
        int hbits = 1;
        while ((1ll << hbits) < 2ll * (ns + T)) hbits++;
        const size_t hbytes = sizeof(unsigned long long) << hbits;
        const bool in_smem = hbytes <= 128 * 1024;
        if (!in_smem && cwb_alloc((void**)&gtab, hbytes * (size_t)K, s) != cudaSuccess)
            return cwb_set_error(ctx, CWB_ENOMEM, "cwb_init: distinct-value table allocation failed");
        if (in_smem) cudaFuncSetAttribute(k_distinct, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hbytes);
        k_distinct<<<K, T, in_smem ? hbytes : 0, s>>>(x, n, ns, hbits, gtab, nsk, st);
        if (gtab) cwb_release(gtab, s);
        if (ctx) ctx->launches++;
    }
    k_design<<<K, 256, 0, s>>>(lo, hi, ns, nsk, z, bnd, st);
    // I3: contiguous row ranges, ~4 waves of 256-thread blocks over all learners (each block
    // stages the learner's boundaries once)
    const int gx = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (32LL * nsm + K - 1) / K));
    dim3 grid(gx, K);
    size_t smem = sizeof(double) * (size_t)(ns > 1 ? ns - 1 : 1);
    const bool use_smem = smem <= 48 * 1024;
    if (!use_smem) smem = 0;
    if (idx_bytes == 1) {
        if (use_smem) k_bin<uint8_t, true><<<grid, 256, smem, s>>>(x, n, ns, bnd, lo, hi, nsk, (uint8_t*)idx, st);
        else k_bin<uint8_t, false><<<grid, 256, 0, s>>>(x, n, ns, bnd, lo, hi, nsk, (uint8_t*)idx, st);
    } else {
        if (use_smem) k_bin<uint16_t, true><<<grid, 256, smem, s>>>(x, n, ns, bnd, lo, hi, nsk, (uint16_t*)idx, st);
        else k_bin<uint16_t, false><<<grid, 256, 0, s>>>(x, n, ns, bnd, lo, hi, nsk, (uint16_t*)idx, st);
    }
    if (ctx) ctx->launches += 4;
    return cwb_check_launch(ctx, "binning kernels");
}

int cwb_launch_init(cwb_ctx* c, const double* X, cudaStream_t s) {
    const int K = c->K, ns = c->n_star, d = c->d;
    int rc = cwb_launch_bin_only(c, c->d_status, X, c->n, K, ns, c->lo, c->hi, c->z, c->bnd, c->idx,
                                 c->idx_bytes, s, c->nsk);
    if (rc) return rc;
    rc = cwb_launch_csr(c, c->idx, c->idx_bytes, c->n, K, ns, c->cnt, c->off, c->perm,
                        c->perm_bytes, s);
    if (rc) return rc;
    if (!c->nb) {
        rc = cwb_fused_plan(c, s);
        if (rc) return rc;
    }
    k_basis<<<K, 128, sizeof(int32_t) * ns, s>>>(c->z, c->lo, c->hi, ns, c->nsk, c->degree, c->n_knots, d,
                                                 c->Zb, c->zj0, c->Zs, c->lwin, c->d_status);
    if (c->nb) {  // unbinned learners: G = Z^T Z on the raw x (cwb_nb.cu)
        rc = cwb_nb_init(c, X, s);
        if (rc) return rc;
    } else {
        k_gram<<<K, 256, 0, s>>>(c->Zb, c->cnt, ns, d, c->lwin, c->G, c->d_status);
    }
    k_lambda<<<K, 32, 0, s>>>(c->G, d, c->df, c->df_kind, c->lambda, c->Ainv, c->Cb, c->d_status);
    k_zt<<<K, 256, 0, s>>>(c->Zb, c->lwin, ns, d, c->W, c->ZT, c->d_status);
    c->launches += 4;
    return cwb_check_launch(c, "pool kernels");
}

// HCWB training-row tables: G_tr = Zb^T diag(cnt_tr) Zb and (G_tr + lambda D)^-1
int cwb_launch_masked_pool(cwb_ctx* c, const uint8_t* mask, uint32_t* cnt_tr, double* G_tr, double* Ainv_tr,
                           cudaStream_t s, double* Cb_tr) {
    const int K = c->K, ns = c->n_star, d = c->d;
    cudaMemsetAsync(cnt_tr, 0, sizeof(uint32_t) * (size_t)K * ns, s);
    const int gx = (int)std::min<int64_t>(64, (c->n + 1023) / 1024);
    const size_t smem = sizeof(uint32_t) * ns;
    if (c->idx_bytes == 1)
        k_count_masked<uint8_t><<<dim3(gx, K), 1024, smem, s>>>((const uint8_t*)c->idx, mask, c->n, ns, cnt_tr,
                                                                c->d_status);
    else
        k_count_masked<uint16_t><<<dim3(gx, K), 1024, smem, s>>>((const uint16_t*)c->idx, mask, c->n, ns, cnt_tr,
                                                                 c->d_status);
    k_gram<<<K, 256, 0, s>>>(c->Zb, cnt_tr, ns, d, c->lwin, G_tr, c->d_status);
    k_inverse_fixed<<<K, 32, 0, s>>>(G_tr, c->lambda, d, Ainv_tr, c->d_status, Cb_tr);
    c->launches += 3;
    return cwb_check_launch(c, "masked pool kernels");
}
