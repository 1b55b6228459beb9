// cwb_iter.cu -- general per-iteration kernels: any n,
// any B, residuals kept row-major (n x Bp, one column per replication) so
// that every gather of a residual row is one coalesced 256-byte segment for
// 32 replications.  Used by cwb_find_best, by cwb_train when the fused
// kernel's shared-memory working set does not fit, and by the stand-alone
// binMatVec primitive.
//
//   k_center   f0 = mean(y), r = y - f0, r^T r      (I8)
//   k_tr_in    Y[B][n] -> Rt[n][Bp]  (tiled transpose)
//   k_h1       u_k(l)[b] = sum_{i in bin l} Rt[i][b]          binMatVec loop
//   k_h234     s = Zb^T u, theta = A^-1 s, delta = 2 theta^T s - theta^T G theta
//   k_h5       k* = argmax delta (lowest k), log, theta_agg += nu theta*   P:L292
//   k_zhat     nu Zb_{k*} theta* at the design points
//   k_h6       r -= zhat[idx_{k*}(i)], partial r^T r
//   k_rr       r^T r per replication, risk log
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <numeric>

#include "cwb_internal.cuh"

namespace {

constexpr int kRowsH6 = 256;  // rows per block in k_h6

// Column reductions over the n rows of each vector (I8): blocks of kColRows rows
// write partial sums, k_center_fin adds them in block order (deterministic).
constexpr int kColRows = 8192;

__global__ void k_colsum(const double* __restrict__ Y, int64_t n, const double* __restrict__ f0, bool sq,
                         double* __restrict__ part, int* status, const uint8_t* mask = nullptr, int keep = 0) {
    const int b = blockIdx.y;
    const double* y = Y + (size_t)b * n;
    const int64_t r0 = (int64_t)blockIdx.x * kColRows, r1 = min(n, r0 + kColRows);
    const double c = f0 ? f0[b] : 0.0;
    double s = 0.0;
    bool bad = false;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
        const double v = y[i];
        bad |= !isfinite(v);
        if (mask && mask[i] != keep) continue;
        const double t = v - c;
        s += sq ? t * t : v;
    }
    if (bad) cwb_dev_fail(status, CWB_ENONFINITE);
    __shared__ double red[32];
    s = warp_sum(s);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0) red[w] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int q = 0; q < nw; q++) t += red[q];
        part[(size_t)b * gridDim.x + blockIdx.x] = t;
    }
}

// mode 0: out[b] = sum / n (mean, also written to offset_out); mode 1: out[b] = sum
__global__ void k_center_fin(const double* __restrict__ part, int nblk, int B, int64_t n, int mode,
                             double* __restrict__ out, double* offset_out, const double* ncount = nullptr) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    double t = 0.0;
    for (int q = 0; q < nblk; q++) t += part[(size_t)b * nblk + q];
    if (mode == 0) {
        t = t / (ncount ? *ncount : (double)n);
        if (offset_out) offset_out[b] = t;
    }
    out[b] = t;
}

// Rt[i][b] = w_i (Y[b][i] - off[b]) for b < B, 0 for the padding columns
__global__ void k_tr_in(const double* __restrict__ Y, int64_t n, int B, int Bp,
                        const double* __restrict__ off, const double* __restrict__ w,
                        double* __restrict__ Rt) {
    __shared__ double tile[32][33];
    const int64_t i0 = (int64_t)blockIdx.x * 32;
    const int b0 = blockIdx.y * 32;
    for (int q = threadIdx.y; q < 32; q += blockDim.y) {  // read rows of Y (contiguous in i)
        const int b = b0 + q;
        const int64_t i = i0 + threadIdx.x;
        double v = 0.0;
        if (b < B && i < n) {
            v = Y[(size_t)b * n + i] - (off ? off[b] : 0.0);
            if (w) v = w[i] * v;
        }
        tile[q][threadIdx.x] = v;
    }
    __syncthreads();
    for (int q = threadIdx.y; q < 32; q += blockDim.y) {  // write rows of Rt (contiguous in b)
        const int64_t i = i0 + q;
        if (i < n) Rt[(size_t)i * Bp + b0 + threadIdx.x] = tile[threadIdx.x][q];
    }
}

// H1: one warp per (learner, bin), lane = replication column; rows of the bin
// in increasing order (the order of the paper's loop over i).
// (fold != NULL: CV folds, rows of column b's own fold colfold[b] >= 0 count as 0)
template <typename PermT>
__global__ void k_h1(const double* __restrict__ Rt, int64_t n, int Bp, int K, int ns,
                     const int32_t* __restrict__ off, const PermT* __restrict__ perm,
                     double* __restrict__ U, const uint8_t* __restrict__ fold = nullptr,
                     const int32_t* __restrict__ colfold = nullptr) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + w;
    if (g >= (int64_t)K * ns) return;
    const int k = (int)(g / ns), l = (int)(g - (int64_t)k * ns);
    const int b = blockIdx.y * 32 + lane;
    const int32_t a0 = off[(size_t)k * (ns + 1) + l], a1 = off[(size_t)k * (ns + 1) + l + 1];
    const PermT* pk = perm + (size_t)k * n;
    const double* col = Rt + b;
    double acc = 0.0;
    int32_t q = a0;
    if (fold) {  // weighted binMatVec (P:L898-904 with 0/1 weights)
        const int fb = colfold[b];
        for (; q < a1; q++) {
            const uint32_t i = pk[q];
            const double v = col[(size_t)i * Bp];
            acc += fold[i] == fb ? 0.0 : v;
        }
        U[(size_t)g * Bp + b] = acc;
        return;
    }
    for (; q + 4 <= a1; q += 4) {
        const uint32_t i0 = pk[q], i1 = pk[q + 1], i2 = pk[q + 2], i3 = pk[q + 3];
        const double v0 = col[(size_t)i0 * Bp], v1 = col[(size_t)i1 * Bp];
        const double v2 = col[(size_t)i2 * Bp], v3 = col[(size_t)i3 * Bp];
        acc += v0; acc += v1; acc += v2; acc += v3;
    }
    for (; q < a1; q++) acc += col[(size_t)pk[q] * Bp];
    U[(size_t)g * Bp + b] = acc;
}

// H1 over a chunk of rows [c CR, (c+1) CR): when a 32-column tile of the residual block
// (n x 256 bytes) exceeds L2, the bins are swept chunk by chunk (one launch per chunk) so that
// the K learners' gathers of a chunk hit L2.  The rows of bin l inside chunk c are a contiguous
// piece of the bin's ascending row list: perm[k][cst[(k nch + c) ns + l] ...] with ccnt rows.
// U += the chunk's sums (chunk 0 writes), so every bin sum is added in chunk order.
__global__ void k_h1_chunk_count(const void* __restrict__ idx, int idx_bytes, int64_t n, int ns, int64_t CR,
                                 int nch, uint32_t* __restrict__ cnt) {
    extern __shared__ uint32_t h[];
    const int c = blockIdx.x, k = blockIdx.y;
    for (int l = threadIdx.x; l < ns; l += blockDim.x) h[l] = 0;
    __syncthreads();
    const int64_t r0 = (int64_t)c * CR, r1 = min(n, r0 + CR);
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
        const uint32_t l = idx_bytes == 1 ? ((const uint8_t*)idx)[(size_t)k * n + i]
                                          : ((const uint16_t*)idx)[(size_t)k * n + i];
        atomicAdd(&h[l], 1u);
    }
    __syncthreads();
    for (int l = threadIdx.x; l < ns; l += blockDim.x) cnt[((size_t)k * nch + c) * ns + l] = h[l];
}

__global__ void k_h1_chunk_start(uint32_t* __restrict__ cnt_cst, const int32_t* __restrict__ off, int K, int ns,
                                 int nch) {
    // in place: cnt -> (start, count) pairs packed as start in the first K nch ns words' twin array
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= (int64_t)K * ns) return;
    const int k = (int)(g / ns), l = (int)(g - (int64_t)k * ns);
    uint32_t run = (uint32_t)off[(size_t)k * (ns + 1) + l];
    uint32_t* cst = cnt_cst + (size_t)K * nch * ns;
    for (int c = 0; c < nch; c++) {
        const size_t e = ((size_t)k * nch + c) * ns + l;
        cst[e] = run;
        run += cnt_cst[e];
    }
}

template <typename PermT>
__global__ void k_h1c(const double* __restrict__ Rt, int64_t n, int Bp, int K, int ns, int nch, int c,
                      const uint32_t* __restrict__ ccnt, const PermT* __restrict__ perm, double* __restrict__ U) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + w;
    if (g >= (int64_t)K * ns) return;
    const int k = (int)(g / ns), l = (int)(g - (int64_t)k * ns);
    const int b = blockIdx.y * 32 + lane;
    const size_t e = ((size_t)k * nch + c) * ns + l;
    const uint32_t cnt = ccnt[e], a0 = ccnt[(size_t)K * nch * ns + e], a1 = a0 + cnt;
    const PermT* pk = perm + (size_t)k * n;
    const double* col = Rt + b;
    double acc = 0.0;
    uint32_t q = a0;
    for (; q + 4 <= a1; q += 4) {
        const uint32_t i0 = pk[q], i1 = pk[q + 1], i2 = pk[q + 2], i3 = pk[q + 3];
        const double v0 = col[(size_t)i0 * Bp], v1 = col[(size_t)i1 * Bp];
        const double v2 = col[(size_t)i2 * Bp], v3 = col[(size_t)i3 * Bp];
        acc += v0; acc += v1; acc += v2; acc += v3;
    }
    for (; q < a1; q++) acc += col[(size_t)pk[q] * Bp];
    double* up = U + (size_t)g * Bp + b;
    *up = c == 0 ? acc : *up + acc;
}

// H1, two replication columns per lane (64 per warp, 16-byte gathers): one warp per (learner, bin) as k_h1,
// rows of the bin in increasing order and one accumulator per column, so every sum is added in exactly
// k_h1's order (bitwise the same U).  The bin's row ids are loaded 32 at a time, one per lane (coalesced),
// and broadcast with a shuffle; the row address is one IMAD.WIDE (row * row stride + column base).
// CHUNK: the rows of chunk c only (k_h1c's tables); U += the chunk sums (chunk 0 writes).
// tri_d > 0 (the cross-Gram build): the columns are the K d basis columns of all learners and only the blocks
// k' >= k of the symmetric cross Gram are needed -- a warp whose 64-column tile ends before learner k's own
// columns (k tri_d) exits (the lower blocks are filled by symmetry afterwards)
template <typename PermT, bool CHUNK>
__global__ void __launch_bounds__(256) k_h1w(const double* __restrict__ Rt, int64_t n, int Bp, int K, int ns,
                                             const int32_t* __restrict__ off, const uint32_t* __restrict__ ccnt,
                                             int nch, int c, const PermT* __restrict__ perm, double* __restrict__ U,
                                             int tri_d = 0) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = blockIdx.x * (blockDim.x >> 5) + w;
    if (g >= K * ns) return;
    const int k = g / ns, l = g - k * ns;
    if (tri_d && (int)blockIdx.y * 64 + 64 <= k * tri_d) return;
    const int b = blockIdx.y * 64 + 2 * lane;
    uint32_t q, a1;
    if (CHUNK) {
        const size_t e = ((size_t)k * nch + c) * ns + l;
        q = ccnt[(size_t)K * nch * ns + e];
        a1 = q + ccnt[e];
    } else {
        q = (uint32_t)off[(size_t)k * (ns + 1) + l];
        a1 = (uint32_t)off[(size_t)k * (ns + 1) + l + 1];
    }
    const PermT* pk = perm + (size_t)k * n;
    const unsigned long long base = (unsigned long long)(Rt + b);
    const uint32_t stride = (uint32_t)Bp * 8u;
    double ax = 0.0, ay = 0.0;
    uint32_t mine = q + lane < a1 ? (uint32_t)pk[q + lane] : 0u;
    for (; q < a1; q += 32) {
        const int cnt = (int)min(32u, a1 - q);
        // the next 32 row ids load while these 32 rows are gathered
        const uint32_t nxt = q + 32 + lane < a1 ? (uint32_t)pk[q + 32 + lane] : 0u;
        int j = 0;
        for (; j + 8 <= cnt; j += 8) {
            uint32_t ii[8];
#pragma unroll
            for (int u = 0; u < 8; u++) ii[u] = __shfl_sync(0xffffffffu, mine, j + u);
            double2 v[8];
#pragma unroll
            for (int u = 0; u < 8; u++) v[u] = __ldg((const double2*)(base + (unsigned long long)ii[u] * stride));
#pragma unroll
            for (int u = 0; u < 8; u++) { ax += v[u].x; ay += v[u].y; }
        }
        for (; j + 4 <= cnt; j += 4) {
            const uint32_t i0 = __shfl_sync(0xffffffffu, mine, j), i1 = __shfl_sync(0xffffffffu, mine, j + 1);
            const uint32_t i2 = __shfl_sync(0xffffffffu, mine, j + 2), i3 = __shfl_sync(0xffffffffu, mine, j + 3);
            const double2 v0 = __ldg((const double2*)(base + (unsigned long long)i0 * stride));
            const double2 v1 = __ldg((const double2*)(base + (unsigned long long)i1 * stride));
            const double2 v2 = __ldg((const double2*)(base + (unsigned long long)i2 * stride));
            const double2 v3 = __ldg((const double2*)(base + (unsigned long long)i3 * stride));
            ax += v0.x; ay += v0.y; ax += v1.x; ay += v1.y;
            ax += v2.x; ay += v2.y; ax += v3.x; ay += v3.y;
        }
        for (; j < cnt; j++) {
            const uint32_t i0 = __shfl_sync(0xffffffffu, mine, j);
            const double2 v0 = __ldg((const double2*)(base + (unsigned long long)i0 * stride));
            ax += v0.x; ay += v0.y;
        }
        mine = nxt;
    }
    double2* up = reinterpret_cast<double2*>(U + (size_t)g * Bp + b);
    if (CHUNK && c != 0) {
        const double2 o = *up;
        *up = make_double2(o.x + ax, o.y + ay);
    } else {
        *up = make_double2(ax, ay);
    }
}

// H2-H4 for one learner (blockIdx.x) and 32 replications (blockIdx.y)
// (HCWB: column b uses Ainv2 / G2 when phase[b mod Bph] != 0)
// (row sharding: smode 1 writes s to Sg[k][d][Bp] and stops, smode 2 reads the summed s from Sg)
__global__ void __launch_bounds__(256, 3) k_h234(const double* __restrict__ U, int Bp, int ns, int d,
                       const double* __restrict__ ZT, int W,
                       const int32_t* __restrict__ lwin, const double* __restrict__ Ainv,
                       const double* __restrict__ G, double* __restrict__ theta,
                       double* __restrict__ delta, const double* __restrict__ Ainv2 = nullptr,
                       const double* __restrict__ G2 = nullptr, const int32_t* __restrict__ phase = nullptr,
                       int Bph = 0, double* __restrict__ Sg = nullptr, int smode = 0,
                       const double* __restrict__ Aset = nullptr, const double* __restrict__ Gset = nullptr,
                       const int32_t* __restrict__ colset = nullptr) {
    __shared__ double S[CWB_MAX_D][33], Th[CWB_MAX_D][33], V[CWB_MAX_D][33];
    const int k = blockIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int b = blockIdx.y * 32 + lane;
    const double* ztk = ZT + (size_t)k * W * d;  // window-major basis: ZT[k][x][j] = Zb_k[lb_j + x][j]
    const double* u = U + (size_t)k * ns * Bp + b;
    for (int j = w; j < d; j += nw) {
        double s;
        if (smode == 2) {
            s = Sg[((size_t)k * d + j) * Bp + b];
        } else {
            const int lb = lwin[((size_t)k * d + j) * 2], le = lwin[((size_t)k * d + j) * 2 + 1];
            const double* zt = ztk + j;
            const double* up = u + (size_t)lb * Bp;
            const int len = le - lb;
            s = 0.0;
            int x = 0;
            // sixteen bins' loads in flight (the window is ~4 n* / (n_knots + 1) bins: ~85 at R3), the FMA
            // chain in bin order
            for (; x + 16 <= len; x += 16) {
                double zq[16], uq[16];
#pragma unroll
                for (int q = 0; q < 16; q++) {
                    zq[q] = zt[(x + q) * d];
                    uq[q] = up[(size_t)(x + q) * Bp];
                }
#pragma unroll
                for (int q = 0; q < 16; q++) s = fma(zq[q], uq[q], s);
            }
            for (; x < len; x++) s = fma(zt[x * d], up[(size_t)x * Bp], s);
            if (smode == 1) Sg[((size_t)k * d + j) * Bp + b] = s;
        }
        S[j][lane] = s;
    }
    if (smode == 1) return;  // block-uniform
    __syncthreads();
    const bool set2 = phase && b < 2 * Bph && phase[b >= Bph ? b - Bph : b] != 0;
    // CV folds: column b uses fold colset[b]'s tables (colset[b] < 0: the pool's)
    const int cs = colset ? colset[b] : -1;
    const int K_ = gridDim.x;
    const double* Ai = (cs >= 0 ? Aset + (size_t)cs * K_ * d * d : (set2 ? Ainv2 : Ainv)) + (size_t)k * d * d;
    for (int j = w; j < d; j += nw) {
        double t = 0.0;
        for (int jp = 0; jp < d; jp++) t += Ai[j * d + jp] * S[jp][lane];
        Th[j][lane] = t;
        theta[((size_t)k * d + j) * Bp + b] = t;
    }
    __syncthreads();
    const double* Gk = (cs >= 0 ? Gset + (size_t)cs * K_ * d * d : (set2 ? G2 : G)) + (size_t)k * d * d;
    for (int j = w; j < d; j += nw) {
        double gt = 0.0;
        for (int jp = max(0, j - (CWB_SPW - 1)); jp <= min(d - 1, j + CWB_SPW - 1); jp++)
            gt += Gk[j * d + jp] * Th[jp][lane];
        V[j][lane] = Th[j][lane] * (2.0 * S[j][lane] - gt);
    }
    __syncthreads();
    if (w == 0) {
        double v = 0.0;
        for (int j = 0; j < d; j++) v += V[j][lane];
        delta[(size_t)k * Bp + b] = v;
    }
}

// H5: argmax over learners per replication; theta_agg update; logs
// H5: block (32 columns, 8 warps); warp w scans the learners k = w, w + 8, ... (strict > keeps the lowest k
// of its sequence), the 8 candidates are merged with ties to the lower k -- argmax delta = argmin SSE, lowest k
// on ties; then theta_agg[k*] += nu theta* with the warps over the coefficients
__global__ void __launch_bounds__(256) k_h5(const double* __restrict__ delta, const double* __restrict__ theta,
                     const double* __restrict__ rr, int K, int d, int B, int Bp, double nu, int m,
                     int32_t* __restrict__ kstar, double* __restrict__ agg, int32_t* k_trace,
                     double* sse_trace, int32_t* k_out, double* theta_out, double* sse_out) {
    __shared__ double sb[8][33];
    __shared__ int sk[8][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int b = blockIdx.x * 32 + lane;
    int ks = -1;
    double best = 0.0;
    for (int k = w; k < K; k += 8) {
        const double v = delta[(size_t)k * Bp + b];
        if (ks < 0 || v > best) { best = v; ks = k; }
    }
    sb[w][lane] = best;
    sk[w][lane] = ks;
    __syncthreads();
    if (w == 0) {
        for (int x = 1; x < 8; x++) {
            const int kx = sk[x][lane];
            const double vx = sb[x][lane];
            if (kx >= 0 && (ks < 0 || vx > best || (vx == best && kx < ks))) { best = vx; ks = kx; }
        }
        if (b >= B) ks = 0;
        sk[0][lane] = ks;
        if (b < B) {
            kstar[b] = ks;
            const double sse = rr[b] - best;
            if (k_trace) k_trace[(size_t)m * B + b] = ks;
            if (sse_trace) sse_trace[(size_t)m * B + b] = sse;
            if (k_out) k_out[b] = ks;
            if (sse_out) sse_out[b] = sse;
        } else {
            kstar[b] = 0;
        }
    }
    __syncthreads();
    if (b >= B) return;
    const int kb = sk[0][lane];
    for (int j = w; j < d; j += 8) {
        const double t = theta[((size_t)kb * d + j) * Bp + b];
        if (agg) agg[((size_t)b * K + kb) * d + j] += nu * t;
        if (theta_out) theta_out[(size_t)b * d + j] = t;
    }
}

// nu * Zb_{k*} theta* at the design points, per (design point, replication)
// columns b < B_nu are scaled by nu, columns B_nu <= b < B by nu2
__global__ void k_zhat(const int32_t* __restrict__ kstar, const double* __restrict__ theta,
                       const int32_t* __restrict__ zj0, const double* __restrict__ Zs, int ns, int d,
                       int B, int Bp, double nu, int B_nu, double nu2, double* __restrict__ zhat) {
    const int b = blockIdx.y * 32 + (threadIdx.x & 31);
    const int l = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (l >= ns) return;
    double v = 0.0;
    if (b < B) {
        const int ks = kstar[b];
        const int a = zj0[(size_t)ks * ns + l];
        const double* zs = Zs + ((size_t)ks * ns + l) * CWB_SPW;
        const double* th = theta + (size_t)ks * d * Bp + b;
        v = zs[0] * th[(size_t)a * Bp];
        for (int q = 1; q < CWB_SPW; q++)
            if (a + q < d) v += zs[q] * th[(size_t)(a + q) * Bp];
        v *= b < B_nu ? nu : nu2;
    }
    zhat[(size_t)l * Bp + b] = v;
}

template <typename IdxT>
__global__ void k_h6(double* __restrict__ Rt, int64_t n, int Bp, const int32_t* __restrict__ kstar,
                     const IdxT* __restrict__ idx, const double* __restrict__ zhat,
                     double* __restrict__ part) {
    __shared__ double red[8][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int b = blockIdx.y * 32 + lane;
    const int ks = kstar[b];
    const IdxT* ik = idx + (size_t)ks * n;
    const int64_t r0 = (int64_t)blockIdx.x * kRowsH6;
    const int64_t r1 = min(n, r0 + kRowsH6);
    double acc = 0.0;
    int64_t i = r0 + w;
    for (; i + 24 < r1; i += 32) {  // four rows in flight (the idx -> zhat gathers are dependent loads)
        uint32_t l[4];
        double x[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            l[u] = ik[i + 8 * u];
            x[u] = Rt[(size_t)(i + 8 * u) * Bp + b];
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const double v = x[u] - zhat[(size_t)l[u] * Bp + b];
            Rt[(size_t)(i + 8 * u) * Bp + b] = v;
            acc += v * v;
        }
    }
    for (; i < r1; i += 8) {
        double v = Rt[(size_t)i * Bp + b] - zhat[(size_t)ik[i] * Bp + b];
        Rt[(size_t)i * Bp + b] = v;
        acc += v * v;
    }
    red[w][lane] = acc;
    __syncthreads();
    if (w == 0) {
        double s = 0.0;
        for (int q = 0; q < 8; q++) s += red[q][lane];
        part[(size_t)blockIdx.x * Bp + b] = s;
    }
}

// H6 with the block's CB columns of zhat staged in shared memory ([ns][CB]): k_h6's zhat gathers (a
// different design-point row per replication) made the L1 the busiest unit (79 %, DRAM 58 %, ncu R3).  Here
// the 16 lanes of a half-warp read 16 distinct columns of the staged table (conflict-free) and the residual
// rows stream at HBM rate.  One 1024-thread block per SM; a warp-step covers 32 / CB rows, eight steps in
// flight; r^T r partials per block in fixed order (rows ascending per thread, warps ascending, then the row
// halves of a column for CB = 16).
constexpr int kH6sThreads = 1024;
template <typename IdxT, int CB>
__global__ void __launch_bounds__(kH6sThreads, 1) k_h6s(double* __restrict__ Rt, int64_t n, int Bp,
                                                       const int32_t* __restrict__ kstar,
                                                       const IdxT* __restrict__ idx, const double* __restrict__ zhat,
                                                       int ns, int64_t rpb, double* __restrict__ part) {
    extern __shared__ double zs[];
    __shared__ double red[kH6sThreads / 32][33];
    constexpr int RW = 32 / CB, U = 8;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int cc = lane % CB, rs = lane / CB;
    const int b = blockIdx.y * CB + cc;
    for (int e = tid; e < ns * CB; e += kH6sThreads) {
        const int l = e / CB;
        zs[e] = zhat[(size_t)l * Bp + blockIdx.y * CB + (e - l * CB)];
    }
    const IdxT* ik = idx + (size_t)kstar[b] * n;
    const int64_t r0 = (int64_t)blockIdx.x * rpb, r1 = min(n, r0 + rpb);
    const int64_t stride = (int64_t)(kH6sThreads / 32) * RW;  // rows per block-step
    __syncthreads();
    double acc = 0.0;
    int64_t i = r0 + w * RW + rs;
    for (; i + (U - 1) * stride < r1; i += U * stride) {
        uint32_t l[U];
        double x[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            l[u] = ik[i + u * stride];
            x[u] = Rt[(size_t)(i + u * stride) * Bp + b];
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const double v = x[u] - zs[l[u] * CB + cc];
            Rt[(size_t)(i + u * stride) * Bp + b] = v;
            acc += v * v;
        }
    }
    for (; i < r1; i += stride) {
        const double v = Rt[(size_t)i * Bp + b] - zs[(uint32_t)ik[i] * CB + cc];
        Rt[(size_t)i * Bp + b] = v;
        acc += v * v;
    }
    red[w][lane] = acc;
    __syncthreads();
    if (w == 0) {
        double t = 0.0;
        for (int q = 0; q < kH6sThreads / 32; q++) t += red[q][lane];
        if (CB == 16) t += __shfl_down_sync(0xffffffffu, t, 16);  // row half 1 of column cc after half 0
        if (lane < CB) part[(size_t)blockIdx.x * Bp + b] = t;
    }
}

// r^T r of every column from the row-block partials: block (32 columns, 32 warps), warp w adds the blocks
// q = w + 32 (8 t + u) into accumulator u (eight loads in flight), the eight accumulators in u order, then the
// 32 warp sums in warp order (fixed order: deterministic)
constexpr int kRrThreads = 1024;
__global__ void __launch_bounds__(kRrThreads, 1) k_rr(const double* __restrict__ part, int nblk, int B, int Bp,
                                                   int64_t n, int m, double* __restrict__ rr, double* risk_trace) {
    __shared__ double red[kRrThreads / 32][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = kRrThreads / 32;
    const int b = blockIdx.x * 32 + lane;
    double a[8];
#pragma unroll
    for (int u = 0; u < 8; u++) a[u] = 0.0;
    int q = w;
    for (; q + 7 * nw < nblk; q += 8 * nw) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; u++) v[u] = part[(size_t)(q + u * nw) * Bp + b];
#pragma unroll
        for (int u = 0; u < 8; u++) a[u] += v[u];
    }
#pragma unroll
    for (int u = 0; u < 8; u++)
        if (q + u * nw < nblk) a[u] += part[(size_t)(q + u * nw) * Bp + b];
    double t = a[0];
#pragma unroll
    for (int u = 1; u < 8; u++) t += a[u];
    red[w][lane] = t;
    __syncthreads();
    if (w == 0 && b < B) {
        double s = 0.0;
        for (int x = 0; x < nw; x++) s += red[x][lane];
        rr[b] = s;
        if (risk_trace) risk_trace[(size_t)m * B + b] = s / (2.0 * (double)n);
    }
}

// row sharding: f0[b] = (sum over all ranks' rows) / n, as k_center_fin mode 0
__global__ void k_mean_glob(const double* __restrict__ sum, int B, int64_t n, double* __restrict__ f0,
                            double* offset_out) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const double t = sum[b] / (double)n;
    f0[b] = t;
    if (offset_out) offset_out[b] = t;
}

// row sharding: risk of one iteration from the summed r^T r, as k_rr
__global__ void k_risk(const double* __restrict__ rr, int B, int64_t n, double* __restrict__ risk_row) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < B) risk_row[b] = rr[b] / (2.0 * (double)n);
}

__global__ void k_zero(double* p, size_t cnt) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (size_t)gridDim.x * blockDim.x)
        p[i] = 0.0;
}

// dense projection out[b][j] = sum_l Zb[l][j] U[l][b] (stand-alone binMatVec, any Zb)
__global__ void k_dense_proj(const double* __restrict__ Zb, const double* __restrict__ U, int ns, int d,
                             int B, int Bp, double* __restrict__ out) {
    const int b = blockIdx.y * 32 + (threadIdx.x & 31);
    const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (j >= d || b >= B) return;
    double s = 0.0;
    for (int l = 0; l < ns; l++) s += Zb[(size_t)l * d + j] * U[(size_t)l * Bp + b];
    out[(size_t)b * d + j] = s;
}

// ---------------------------------------------------------------- ACWB path
// Accelerated CWB, Algorithm 2.  Replication b keeps, row-major with one
// column per replication, F = y - f (primary model), H = y - h (momentum model); its
// pseudo residuals r = y - g = (1 - theta_m) F + theta_m H (lines 5-6) and error-corrected
// residuals c (lines 9-13) are the columns b and B + b of Rt, so binMatVec, fit and SSE
// (k_h1, k_h234) run once on the 2B columns.

// per replication: k = argmin SSE of column b (line 7), k_cor of column B + b (line 14),
// traces, parameter bookkeeping of P:L966 (theta_g = (1 - vt) theta_f + vt theta_h,
// theta_f = theta_g + nu e_k theta, theta_h += eta e_kcor theta_cor)
__global__ void k_acwb_select(const double* __restrict__ delta, const double* __restrict__ theta,
                              const double* __restrict__ rr, int K, int d, int B, int Bp, double nu, double vt,
                              double eta, int m, int32_t* __restrict__ kstar, double* __restrict__ tf,
                              double* __restrict__ th, int32_t* k_trace, int32_t* kcor_trace, double* sse_trace) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    int ks = 0, kc = 0;
    double best = delta[b], bestc = delta[B + b];
    for (int k = 1; k < K; k++) {
        const double v = delta[(size_t)k * Bp + b], vc = delta[(size_t)k * Bp + B + b];
        if (v > best) { best = v; ks = k; }
        if (vc > bestc) { bestc = vc; kc = k; }
    }
    kstar[b] = ks;
    kstar[B + b] = kc;
    double* f = tf + (size_t)b * K * d;
    double* h = th + (size_t)b * K * d;
    for (int a = 0; a < K * d; a++) f[a] = (1.0 - vt) * f[a] + vt * h[a];
    for (int j = 0; j < d; j++) {
        f[ks * d + j] += nu * theta[((size_t)ks * d + j) * Bp + b];
        h[kc * d + j] += eta * theta[((size_t)kc * d + j) * Bp + B + b];
    }
    if (k_trace) k_trace[(size_t)m * B + b] = ks;
    if (kcor_trace) kcor_trace[(size_t)m * B + b] = kc;
    if (sse_trace) sse_trace[(size_t)m * B + b] = rr[b] - best;
}

// Rt[i][B + b] = Rt[i][b], F[i][b] = H[i][b] = Rt[i][b] (= y - f0: f = h = g = f0, line 2)
__global__ void k_acwb_init(double* __restrict__ Rt, double* __restrict__ F, double* __restrict__ H, int64_t n,
                            int B, int Bp, int Bq) {
    const int b = blockIdx.y * 32 + (threadIdx.x & 31);
    if (b >= B) return;
    for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n;
         i += (int64_t)gridDim.x * (blockDim.x >> 5)) {
        const double v = Rt[(size_t)i * Bp + b];
        Rt[(size_t)i * Bp + B + b] = v;
        F[(size_t)i * Bq + b] = v;
        H[(size_t)i * Bq + b] = v;
    }
}

// line 8: F = r - nu b_k, line 16: H -= eta b_kcor; then the residuals of iteration m+1:
// r' = (1 - vt1) F + vt1 H, c' = r' + a1 (c - b_kcor) (lines 4-6, 10); row-block partial
// sums of F^2 (risk of f), r'^2 and c'^2 (r^T r of the next fits)
template <typename IdxT>
__global__ void k_acwb_update(double* __restrict__ Rt, double* __restrict__ F, double* __restrict__ H, int64_t n,
                              int B, int Bp, int Bq, const int32_t* __restrict__ kstar, const IdxT* __restrict__ idx,
                              const double* __restrict__ zhat, double eta, double vt1, double a1,
                              double* __restrict__ part) {
    __shared__ double red[3][8][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int b = blockIdx.y * 32 + lane;
    const bool live = b < B;
    const int ks = live ? kstar[b] : 0, kc = live ? kstar[B + b] : 0;
    const IdxT* ik = idx + (size_t)ks * n;
    const IdxT* ic = idx + (size_t)kc * n;
    const int64_t r0 = (int64_t)blockIdx.x * kRowsH6, r1 = min(n, r0 + kRowsH6);
    double sf = 0.0, sr = 0.0, sc = 0.0;
    if (live)
        for (int64_t i = r0 + w; i < r1; i += 8) {
            const double r = Rt[(size_t)i * Bp + b], c = Rt[(size_t)i * Bp + B + b];
            const double bk = zhat[(size_t)ik[i] * Bp + b];        // nu b_k (scaled by k_zhat)
            const double bc = zhat[(size_t)ic[i] * Bp + B + b];    // b_kcor (unscaled)
            const double Fi = r - bk;
            const double Hi = H[(size_t)i * Bq + b] - eta * bc;
            const double rn = (1.0 - vt1) * Fi + vt1 * Hi;
            const double cn = rn + a1 * (c - bc);
            F[(size_t)i * Bq + b] = Fi;
            H[(size_t)i * Bq + b] = Hi;
            Rt[(size_t)i * Bp + b] = rn;
            Rt[(size_t)i * Bp + B + b] = cn;
            sf += Fi * Fi;
            sr += rn * rn;
            sc += cn * cn;
        }
    red[0][w][lane] = sf;
    red[1][w][lane] = sr;
    red[2][w][lane] = sc;
    __syncthreads();
    if (w < 3 && live) {
        double t = 0.0;
        for (int q = 0; q < 8; q++) t += red[w][q][lane];
        part[((size_t)w * gridDim.x + blockIdx.x) * Bq + b] = t;
    }
}

// rr of the next fits (columns b, B + b) and risk of f after iteration m (R_emp = F^T F / (2n))
__global__ void k_acwb_rr(const double* __restrict__ part, int nblk, int B, int Bq, int64_t n, int m,
                          double* __restrict__ rr, double* risk_trace) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    double sf = 0.0, sr = 0.0, sc = 0.0;
    for (int q = 0; q < nblk; q++) {
        sf += part[((size_t)0 * nblk + q) * Bq + b];
        sr += part[((size_t)1 * nblk + q) * Bq + b];
        sc += part[((size_t)2 * nblk + q) * Bq + b];
    }
    rr[b] = sr;
    rr[B + b] = sc;
    if (risk_trace) risk_trace[(size_t)m * B + b] = sf / (2.0 * (double)n);
}

// ---------------------------------------------------------------- HCWB path
// Hybrid CWB, Algorithm 3: per replication, ACWB fitted on the training rows
// (val_mask == 0; their residual columns are zero on validation rows, and they use the
// training-row G_tr, (G_tr + lambda D)^-1) while the validation-risk patience counter is
// below pat0, then CWB on all rows (G, A^-1 of the pool).  phase[b]: 0 ACWB, 1 CWB.

__global__ void k_hcwb_scale_vprev(double* __restrict__ v, const double* __restrict__ cnt, int B) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < B) v[b] = v[b] / (2.0 * cnt[1]);
}

__global__ void k_fill_int(int32_t* __restrict__ p, int cnt, int v) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < cnt) p[b] = v;
}

__global__ void k_mask_count(const uint8_t* __restrict__ mask, int64_t n, double* __restrict__ cnt,
                             int* __restrict__ status) {
    __shared__ double red[32];
    double v = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) v += mask[i] ? 1.0 : 0.0;
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int q = 0; q < (int)(blockDim.x >> 5); q++) t += red[q];
        cnt[0] = (double)n - t;  // training rows
        cnt[1] = t;              // validation rows
        // HCWB needs both sets: the training fits divide by the training rows, the patience rule by the
        // validation rows (Alg. 3)
        if (t == 0.0 || t == (double)n) cwb_dev_fail(status, CWB_EINVAL);
    }
}

// F = H = Rt[i][b] (= y - f0, all rows); fitting columns b, B+b masked to the training rows
__global__ void k_hcwb_init(double* __restrict__ Rt, double* __restrict__ F, double* __restrict__ H,
                            const uint8_t* __restrict__ mask, int64_t n, int B, int Bp, int Bq) {
    const int b = blockIdx.y * 32 + (threadIdx.x & 31);
    if (b >= B) return;
    for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n;
         i += (int64_t)gridDim.x * (blockDim.x >> 5)) {
        const double v = Rt[(size_t)i * Bp + b];
        F[(size_t)i * Bq + b] = v;
        H[(size_t)i * Bq + b] = v;
        const double vm = mask[i] ? 0.0 : v;
        Rt[(size_t)i * Bp + b] = vm;
        Rt[(size_t)i * Bp + B + b] = vm;
    }
}

__global__ void k_hcwb_select(const double* __restrict__ delta, const double* __restrict__ theta,
                              const double* __restrict__ rr, const int32_t* __restrict__ phase, int K, int d, int B,
                              int Bp, double nu, double vt, double eta, int m, int32_t* __restrict__ kstar,
                              double* __restrict__ tf, double* __restrict__ th, int32_t* k_trace, int32_t* kcor_trace,
                              double* sse_trace) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const bool acc = phase[b] == 0;
    int ks = 0, kc = 0;
    double best = delta[b], bestc = delta[B + b];
    for (int k = 1; k < K; k++) {
        const double v = delta[(size_t)k * Bp + b], vc = delta[(size_t)k * Bp + B + b];
        if (v > best) { best = v; ks = k; }
        if (vc > bestc) { bestc = vc; kc = k; }
    }
    kstar[b] = ks;
    kstar[B + b] = kc;
    double* f = tf + (size_t)b * K * d;
    double* h = th + (size_t)b * K * d;
    if (acc) {  // ACWB bookkeeping
        for (int a = 0; a < K * d; a++) f[a] = (1.0 - vt) * f[a] + vt * h[a];
        for (int j = 0; j < d; j++) {
            f[ks * d + j] += nu * theta[((size_t)ks * d + j) * Bp + b];
            h[kc * d + j] += eta * theta[((size_t)kc * d + j) * Bp + B + b];
        }
    } else {    // CWB aggregation
        for (int j = 0; j < d; j++) f[ks * d + j] += nu * theta[((size_t)ks * d + j) * Bp + b];
    }
    if (k_trace) k_trace[(size_t)m * B + b] = ks;
    if (kcor_trace) kcor_trace[(size_t)m * B + b] = acc ? kc : -1;
    if (sse_trace) sse_trace[(size_t)m * B + b] = rr[b] - best;
}

// pass 1: models after iteration m.  ACWB: F = (1-vt)F + vt H - nu b_k (= y - (g + nu b_k)),
// H -= eta b_kcor; CWB: F -= nu b_k.  Partial sums of F^2 on all rows and on validation rows.
template <typename IdxT>
__global__ void k_hcwb_update(double* __restrict__ F, double* __restrict__ H, const uint8_t* __restrict__ mask,
                              int64_t n, int B, int Bp, int Bq, const int32_t* __restrict__ phase,
                              const int32_t* __restrict__ kstar, const IdxT* __restrict__ idx,
                              const double* __restrict__ zhat, double vt, double eta, double* __restrict__ part) {
    __shared__ double red[2][8][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int b = blockIdx.y * 32 + lane;
    const bool live = b < B;
    const bool acc = live && phase[b] == 0;
    const int ks = live ? kstar[b] : 0, kc = live ? kstar[B + b] : 0;
    const IdxT* ik = idx + (size_t)ks * n;
    const IdxT* ic = idx + (size_t)kc * n;
    const int64_t r0 = (int64_t)blockIdx.x * kRowsH6, r1 = min(n, r0 + kRowsH6);
    double sa = 0.0, sv = 0.0;
    if (live)
        for (int64_t i = r0 + w; i < r1; i += 8) {
            const double Fo = F[(size_t)i * Bq + b];
            const double bk = zhat[(size_t)ik[i] * Bp + b];
            double Fn;
            if (acc) {
                const double Ho = H[(size_t)i * Bq + b];
                const double bc = zhat[(size_t)ic[i] * Bp + B + b];
                Fn = (1.0 - vt) * Fo + vt * Ho - bk;
                H[(size_t)i * Bq + b] = Ho - eta * bc;
            } else {
                Fn = Fo - bk;
            }
            F[(size_t)i * Bq + b] = Fn;
            sa += Fn * Fn;
            if (mask[i]) sv += Fn * Fn;
        }
    red[0][w][lane] = sa;
    red[1][w][lane] = sv;
    __syncthreads();
    if (w < 2 && live) {
        double t = 0.0;
        for (int q = 0; q < 8; q++) t += red[w][q][lane];
        part[((size_t)w * gridDim.x + blockIdx.x) * Bq + b] = t;
    }
}

// risk traces and the patience counter (Alg. 3 line 6): phase 0 -> 1 after pat0 consecutive
// increases of the validation risk
__global__ void k_hcwb_decide(const double* __restrict__ part, int nblk, int B, int Bq, int64_t n,
                              const double* __restrict__ cnt, int m, int pat0, int32_t* __restrict__ phase,
                              int32_t* __restrict__ pat, double* __restrict__ vprev, int32_t* switch_iter,
                              double* risk_trace, double* val_risk_trace) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    double sa = 0.0, sv = 0.0;
    for (int q = 0; q < nblk; q++) {
        sa += part[((size_t)0 * nblk + q) * Bq + b];
        sv += part[((size_t)1 * nblk + q) * Bq + b];
    }
    const double vr = sv / (2.0 * cnt[1]);
    if (risk_trace) risk_trace[(size_t)m * B + b] = sa / (2.0 * (double)n);
    if (val_risk_trace) val_risk_trace[(size_t)m * B + b] = vr;
    if (phase[b] == 0) {
        pat[b] = vr > vprev[b] ? pat[b] + 1 : 0;
        if (pat[b] >= pat0) {
            phase[b] = 1;
            if (switch_iter) switch_iter[b] = m + 1;
        }
    }
    vprev[b] = vr;
}

// pass 2: fitting columns of iteration m+1.  ACWB: r' = (1-vt1) F + vt1 H, c' = r' + a1 (c - b_kcor),
// zero on validation rows; CWB: r' = F on all rows, c' = 0.  Partial sums of r'^2, c'^2.
template <typename IdxT>
__global__ void k_hcwb_prepare(double* __restrict__ Rt, const double* __restrict__ F, const double* __restrict__ H,
                               const uint8_t* __restrict__ mask, int64_t n, int B, int Bp, int Bq,
                               const int32_t* __restrict__ phase, const int32_t* __restrict__ kstar,
                               const IdxT* __restrict__ idx, const double* __restrict__ zhat, double vt1, double a1,
                               double* __restrict__ part) {
    __shared__ double red[2][8][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int b = blockIdx.y * 32 + lane;
    const bool live = b < B;
    const bool acc = live && phase[b] == 0;
    const int kc = live ? kstar[B + b] : 0;
    const IdxT* ic = idx + (size_t)kc * n;
    const int64_t r0 = (int64_t)blockIdx.x * kRowsH6, r1 = min(n, r0 + kRowsH6);
    double sr = 0.0, sc = 0.0;
    if (live)
        for (int64_t i = r0 + w; i < r1; i += 8) {
            const double Fi = F[(size_t)i * Bq + b];
            double rn, cn;
            if (acc) {
                rn = (1.0 - vt1) * Fi + vt1 * H[(size_t)i * Bq + b];
                cn = rn + a1 * (Rt[(size_t)i * Bp + B + b] - zhat[(size_t)ic[i] * Bp + B + b]);
                if (mask[i]) { rn = 0.0; cn = 0.0; }
            } else {
                rn = Fi;
                cn = 0.0;
            }
            Rt[(size_t)i * Bp + b] = rn;
            Rt[(size_t)i * Bp + B + b] = cn;
            sr += rn * rn;
            sc += cn * cn;
        }
    red[0][w][lane] = sr;
    red[1][w][lane] = sc;
    __syncthreads();
    if (w < 2 && live) {
        double t = 0.0;
        for (int q = 0; q < 8; q++) t += red[w][q][lane];
        part[((size_t)(2 + w) * gridDim.x + blockIdx.x) * Bq + b] = t;
    }
}

__global__ void k_hcwb_rr(const double* __restrict__ part, int nblk, int B, int Bq, double* __restrict__ rr) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    double sr = 0.0, sc = 0.0;
    for (int q = 0; q < nblk; q++) {
        sr += part[((size_t)2 * nblk + q) * Bq + b];
        sc += part[((size_t)3 * nblk + q) * Bq + b];
    }
    rr[b] = sr;
    rr[B + b] = sc;
}

// ---------------------------------------------------------------- Bernoulli loss
// CWB (Alg. 1 supp.) with the Bernoulli loss L(y, f) = log(1 + exp(f)) - y f,
// y in {0, 1}: offset logit(mean y) (line 2), pseudo residuals
// r = y - 1 / (1 + exp(-f)) (line 4); the base-learner fits and the selection are
// the L2 fits of r as for the L2 loss.  Per replication the fit F[i][b] = f(x_i) and the
// targets Yt[i][b] are kept row-major next to the residuals Rt[i][b].

// f0[b] = log(p / (1 - p)), p = mean(y_b) (in f0 on entry); CWB_EDEGENERATE for p in {0, 1}
__global__ void k_bern_offset(double* __restrict__ f0, int B, double* offset_out, int* status) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const double p = f0[b];
    if (!(p > 0.0 && p < 1.0)) cwb_dev_fail(status, CWB_EDEGENERATE);
    const double t = log(p / (1.0 - p));
    f0[b] = t;
    if (offset_out) offset_out[b] = t;
}

// Yt = Y^T (0/1 check, CWB_EINVAL otherwise); padding columns 0
__global__ void k_bern_init(const double* __restrict__ Y, int64_t n, int B, int Bp, double* __restrict__ Yt,
                            int* status) {
    __shared__ double tile[32][33];
    const int64_t i0 = (int64_t)blockIdx.x * 32;
    const int b0 = blockIdx.y * 32;
    for (int q = threadIdx.y; q < 32; q += blockDim.y) {
        const int b = b0 + q;
        const int64_t i = i0 + threadIdx.x;
        double v = 0.0;
        if (b < B && i < n) {
            v = Y[(size_t)b * n + i];
            if (v != 0.0 && v != 1.0) cwb_dev_fail(status, CWB_EINVAL);
        }
        tile[q][threadIdx.x] = v;
    }
    __syncthreads();
    for (int q = threadIdx.y; q < 32; q += blockDim.y) {
        const int64_t i = i0 + q;
        const int b = b0 + threadIdx.x;
        if (i < n) Yt[(size_t)i * Bp + b] = tile[threadIdx.x][q];
    }
}

// (f0 != NULL) f = f0 (line 2); (zhat != NULL) f += nu b_{k*}(x) at the design points (line 10);
// then r = y - sigma(f) (line 4 of the next iteration) and row-block partial sums of r^2, L(y, f)
template <typename IdxT>
__global__ void k_bern_update(double* __restrict__ Rt, double* __restrict__ F, const double* __restrict__ Yt,
                              int64_t n, int Bp, int B, const double* __restrict__ f0, const int32_t* __restrict__ kstar,
                              const IdxT* __restrict__ idx, const double* __restrict__ zhat, double* __restrict__ part,
                              int nblk) {
    __shared__ double red[2][8][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int b = blockIdx.y * 32 + lane;
    const IdxT* ik = zhat ? idx + (size_t)kstar[b] * n : nullptr;
    const int64_t r0 = (int64_t)blockIdx.x * kRowsH6;
    const int64_t r1 = min(n, r0 + kRowsH6);
    double a2 = 0.0, al = 0.0;
    for (int64_t i = r0 + w; i < r1; i += 8) {
        const size_t e = (size_t)i * Bp + b;
        double f;
        if (f0) {
            f = b < B ? f0[b] : 0.0;
            F[e] = f;
        } else {
            f = F[e];
        }
        if (zhat) {
            f = f + zhat[(size_t)ik[i] * Bp + b];
            F[e] = f;
        }
        const double y = Yt[e];
        double lo;
        const double r = bern_resid(y, f, &lo);
        Rt[e] = r;
        a2 += r * r;
        al += lo;
    }
    red[0][w][lane] = a2;
    red[1][w][lane] = al;
    __syncthreads();
    if (w == 0) {
        double s2 = 0.0, sl = 0.0;
        for (int q = 0; q < 8; q++) { s2 += red[0][q][lane]; sl += red[1][q][lane]; }
        part[(size_t)blockIdx.x * Bp + b] = s2;
        part[((size_t)nblk + blockIdx.x) * Bp + b] = sl;
    }
}

// rr[b] = r^T r; risk_trace[m][b] = mean L(y, f) (m >= 0)
__global__ void k_bern_rr(const double* __restrict__ part, int nblk, int B, int Bp, int64_t n, int m,
                          double* __restrict__ rr, double* risk_trace) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    double s = 0.0, l = 0.0;
    for (int q = 0; q < nblk; q++) {
        s += part[(size_t)q * Bp + b];
        l += part[((size_t)nblk + q) * Bp + b];
    }
    rr[b] = s;
    if (risk_trace && m >= 0) risk_trace[(size_t)m * B + b] = l / (double)n;
}

// ---------------------------------------------------------------- CV folds
// CWB with 0/1 observation weights per replication: column b fits on the rows
// whose fold differs from colfold[b] (colfold[b] = -1: every row).

// per column (one block): f0 = mean of y over the training rows, rr = their sum of (y - f0)^2,
// training / held-out row counts; argument checks (CWB_EINVAL)
__global__ void k_fold_stats(const double* __restrict__ Y, int64_t n, const uint8_t* __restrict__ fold, int F,
                             const int32_t* __restrict__ colfold, double* __restrict__ f0, double* __restrict__ rr,
                             double* __restrict__ ntr, double* __restrict__ nho, double* offset_out, int* status) {
    __shared__ double red[3][32];
    const int b = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int fb = colfold[b];
    if (fb >= F || fb < -1) cwb_dev_fail(status, CWB_EINVAL);
    const double* y = Y + (size_t)b * n;
    double sy = 0.0, c = 0.0;
    bool bad = false, badf = false;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double v = y[i];
        bad |= !isfinite(v);
        badf |= fold[i] >= F;
        if (fold[i] != fb) { sy += v; c += 1.0; }
    }
    if (bad) cwb_dev_fail(status, CWB_ENONFINITE);
    if (badf) cwb_dev_fail(status, CWB_EINVAL);
    sy = warp_sum(sy);
    c = warp_sum(c);
    if (lane == 0) { red[0][w] = sy; red[1][w] = c; }
    __syncthreads();
    double ts = 0.0, tc = 0.0;
    for (int q = 0; q < nw; q++) { ts += red[0][q]; tc += red[1][q]; }
    if (tc == 0.0) { if (threadIdx.x == 0) cwb_dev_fail(status, CWB_EINVAL); return; }
    const double m = ts / tc;
    double s2 = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
        if (fold[i] != fb) { const double e = y[i] - m; s2 += e * e; }
    s2 = warp_sum(s2);
    if (lane == 0) red[2][w] = s2;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int q = 0; q < nw; q++) t += red[2][q];
        f0[b] = m;
        rr[b] = t;
        ntr[b] = tc;
        nho[b] = (double)n - tc;
        if (offset_out) offset_out[b] = m;
    }
}

__global__ void k_fold_mask(const uint8_t* __restrict__ fold, int64_t n, int f, uint8_t* __restrict__ mask) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        mask[i] = fold[i] == f ? 1 : 0;
}

// r -= zhat[idx_k*(i)] on every row; partials of r^2 over the training and the held-out rows
template <typename IdxT>
__global__ void k_h6_fold(double* __restrict__ Rt, int64_t n, int Bp, const int32_t* __restrict__ kstar,
                          const IdxT* __restrict__ idx, const double* __restrict__ zhat,
                          const uint8_t* __restrict__ fold, const int32_t* __restrict__ colfold, int B,
                          double* __restrict__ part, int nblk) {
    __shared__ double red[2][8][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int b = blockIdx.y * 32 + lane;
    const int ks = kstar[b];
    const int fb = b < B ? colfold[b] : -1;
    const IdxT* ik = idx + (size_t)ks * n;
    const int64_t r0 = (int64_t)blockIdx.x * kRowsH6;
    const int64_t r1 = min(n, r0 + kRowsH6);
    double at = 0.0, ah = 0.0;
    for (int64_t i = r0 + w; i < r1; i += 8) {
        const double v = Rt[(size_t)i * Bp + b] - zhat[(size_t)ik[i] * Bp + b];
        Rt[(size_t)i * Bp + b] = v;
        if (fold[i] == fb) ah += v * v;
        else at += v * v;
    }
    red[0][w][lane] = at;
    red[1][w][lane] = ah;
    __syncthreads();
    if (w < 2) {
        double t = 0.0;
        for (int q = 0; q < 8; q++) t += red[w][q][lane];
        part[((size_t)w * nblk + blockIdx.x) * Bp + b] = t;
    }
}

// rr[b] = training r^T r; risk_trace = rr / (2 n_train), val_risk_trace = held-out / (2 n_held) (0: none)
__global__ void k_rr_fold(const double* __restrict__ part, int nblk, int B, int Bp, const double* __restrict__ ntr,
                          const double* __restrict__ nho, int m, double* __restrict__ rr, double* risk_trace,
                          double* val_risk_trace) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    double st = 0.0, sh = 0.0;
    for (int q = 0; q < nblk; q++) {
        st += part[(size_t)q * Bp + b];
        sh += part[((size_t)nblk + q) * Bp + b];
    }
    rr[b] = st;
    if (risk_trace) risk_trace[(size_t)m * B + b] = st / (2.0 * ntr[b]);
    if (val_risk_trace) val_risk_trace[(size_t)m * B + b] = nho[b] > 0.0 ? sh / (2.0 * nho[b]) : 0.0;
}

// ---------------------------------------------------------------- learner sharding
// (include/cwb.h cwb_attach_comm_learners, SURVEY 8(e) alternative): rank r fits the learners
// [k0, k1); per replication its best (delta, k, theta) goes to slot r of buf[world][Bp][d + 2]
// (zeros elsewhere), a sum all-reduce gathers the slots, and every rank takes the best over the
// slots in rank order (= k order: strict > keeps the lowest k on ties), then the H5 bookkeeping.
__global__ void k_lshard_pack(const double* __restrict__ delta, const double* __restrict__ theta, int k0, int k1,
                              int d, int B, int Bp, int rank, double* __restrict__ buf) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    int ks = k0;
    double best = delta[(size_t)k0 * Bp + b];
    for (int k = k0 + 1; k < k1; k++) {
        const double v = delta[(size_t)k * Bp + b];
        if (v > best) { best = v; ks = k; }
    }
    double* o = buf + ((size_t)rank * Bp + b) * (d + 2);
    o[0] = best;
    o[1] = (double)ks;
    for (int j = 0; j < d; j++) o[2 + j] = theta[((size_t)ks * d + j) * Bp + b];
}

__global__ void k_lshard_pick(const double* __restrict__ buf, int world, const double* __restrict__ rr, int K, int d,
                              int B, int Bp, double nu, int m, int32_t* __restrict__ kstar, double* __restrict__ theta,
                              double* __restrict__ agg, int32_t* k_trace, double* sse_trace, int32_t* k_out,
                              double* theta_out, double* sse_out) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= Bp) return;
    if (b >= B) { kstar[b] = 0; return; }
    int rb = 0;
    double best = buf[(size_t)b * (d + 2)];
    for (int r = 1; r < world; r++) {
        const double v = buf[((size_t)r * Bp + b) * (d + 2)];
        if (v > best) { best = v; rb = r; }
    }
    const double* o = buf + ((size_t)rb * Bp + b) * (d + 2);
    const int ks = (int)o[1];
    kstar[b] = ks;
    for (int j = 0; j < d; j++) theta[((size_t)ks * d + j) * Bp + b] = o[2 + j];
    const double sse = rr[b] - best;
    if (agg)
        for (int j = 0; j < d; j++) agg[((size_t)b * K + ks) * d + j] += nu * o[2 + j];
    if (k_trace) k_trace[(size_t)m * B + b] = ks;
    if (sse_trace) sse_trace[(size_t)m * B + b] = sse;
    if (k_out) k_out[b] = ks;
    if (sse_out) sse_out[b] = sse;
    if (theta_out)
        for (int j = 0; j < d; j++) theta_out[(size_t)b * d + j] = o[2 + j];
}

// ---------------------------------------------------------------- narrow path
// binMatVec sums for a few residual vectors (B <= 4), e.g. one
// findBestBaselearner on a single residual: HBM-bound on the index vector.  A CTA
// stages a chunk of the residual rows in shared memory; each warp streams one
// learner's index vector over the chunk (coalesced), groups the lanes holding the
// same bin (__match_any_sync), and the lowest lane of each group adds the group's
// values, in lane order, into the warp's private histogram (distinct bins: no
// conflicting writes, no atomics, deterministic).  Histograms of the row ranges go
// to P[range][k][l][q] and are combined in range order by k_narrow_combine.
// TMA bulk copies (cp.async.bulk, global -> shared) completing on an mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Staged chunk of residual rows (NB columns) and of the index slices of the CTA's LPC
// learners.  TMA = true: 16-byte aligned chunks, one elected thread issues the bulk copies
// of chunk j+1 while chunk j is processed (double buffer); otherwise plain loads.
template <typename IdxT, int NB, bool TMA>
__global__ void __launch_bounds__(256) k_h1_narrow(const double* __restrict__ R, int64_t n, int K, int ns,
                                                    const IdxT* __restrict__ idx, int64_t rows_per_cta, int nc,
                                                    double* __restrict__ P) {
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) uint64_t bars[2];
    const int T = blockDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, LPC = T >> 5;
    const int NBUF = TMA ? 2 : 1;
    const size_t buf_bytes = sizeof(double) * (size_t)nc * NB + sizeof(IdxT) * (size_t)LPC * nc;  // 16-multiple
    double* hist = (double*)((unsigned char*)sm + NBUF * buf_bytes) + (size_t)warp * ns * NB;
    const int k0 = blockIdx.y * LPC, k = k0 + warp;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta, r1 = min(n, r0 + rows_per_cta);
    const int nchunks = (int)((r1 - r0 + nc - 1) / nc);
    for (int a = lane; a < ns * NB; a += 32) hist[a] = 0.0;
    auto rs_of = [&](int buf) { return (double*)((unsigned char*)sm + buf * buf_bytes); };
    auto is_of = [&](int buf) { return (IdxT*)(rs_of(buf) + (size_t)nc * NB); };
    // TMA: rows of the chunk copied in 16-byte units; residual tail rows (len % 2) by plain loads
    auto issue = [&](int j) {
        const int buf = j & 1;
        const int64_t c0 = r0 + (int64_t)j * nc;
        const int len = (int)min((int64_t)nc, r1 - c0);
        const uint32_t rbytes = (uint32_t)((len * sizeof(double)) & ~(size_t)15);
        const uint32_t ibytes = (uint32_t)((len * sizeof(IdxT) + 15) & ~(size_t)15);  // idx buffer has slack
        int nl = min(LPC, K - k0);
        mbar_expect_tx(&bars[buf], NB * rbytes + nl * ibytes);
        for (int q = 0; q < NB; q++)
            if (rbytes) bulk_g2s(rs_of(buf) + (size_t)q * nc, R + (size_t)q * n + c0, rbytes, &bars[buf]);
        for (int w = 0; w < nl; w++)
            bulk_g2s(is_of(buf) + (size_t)w * nc, idx + (size_t)(k0 + w) * n + c0, ibytes, &bars[buf]);
    };
    if (TMA) {
        if (tid == 0) {
            mbar_init(&bars[0], 1);
            mbar_init(&bars[1], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (tid == 0 && nchunks > 0) issue(0);
    }
    for (int j = 0; j < nchunks; j++) {
        const int buf = TMA ? (j & 1) : 0;
        const int64_t c0 = r0 + (int64_t)j * nc;
        const int len = (int)min((int64_t)nc, r1 - c0);
        double* rs = rs_of(buf);
        IdxT* is = is_of(buf);
        if (TMA) {
            if (tid == 0 && j + 1 < nchunks) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(j + 1);
            }
            const int rt = len & 1;  // residual rows not covered by the 16-byte copy
            if (rt && tid < NB) rs[(size_t)tid * nc + len - 1] = __ldg(R + (size_t)tid * n + c0 + len - 1);
            mbar_wait(&bars[buf], (uint32_t)((j >> 1) & 1));
            if (rt) __syncthreads();
        } else {
            __syncthreads();  // previous chunk consumed
            for (int q = 0; q < NB; q++)
                for (int i = tid; i < len; i += T) rs[(size_t)q * nc + i] = __ldg(R + (size_t)q * n + c0 + i);
            for (int w = 0; w < LPC; w++) {
                const IdxT* src = idx + (size_t)min(k0 + w, K - 1) * n + c0;
#pragma unroll 4
                for (int i = tid; i < len; i += T) is[w * nc + i] = __ldg(src + i);
            }
            __syncthreads();
        }
        if (k < K) {
            const IdxT* iw = is + warp * nc;
            constexpr int U4 = 4;  // warp-steps in flight: loads and MATCHes of 4 steps overlap
            for (int i0 = 0; i0 < len; i0 += 32 * U4) {
                uint32_t bin[U4];
                unsigned peers[U4];
                double v[U4][NB], sum[U4][NB];
#pragma unroll
                for (int u = 0; u < U4; u++) {
                    const int i = i0 + u * 32 + lane;
                    const bool valid = i < len;
                    bin[u] = valid ? (uint32_t)iw[i] : 0xffffffffu;
#pragma unroll
                    for (int q = 0; q < NB; q++) { v[u][q] = valid ? rs[(size_t)q * nc + i] : 0.0; sum[u][q] = v[u][q]; }
                }
#pragma unroll
                for (int u = 0; u < U4; u++) peers[u] = __match_any_sync(0xffffffffu, bin[u]);
                // group sums in lane order, led by the lowest lane of each group
                unsigned rem[U4];
                bool lead[U4];
#pragma unroll
                for (int u = 0; u < U4; u++) {
                    lead[u] = bin[u] != 0xffffffffu && (peers[u] & ((1u << lane) - 1u)) == 0u;
                    rem[u] = lead[u] ? (peers[u] & (peers[u] - 1u)) : 0u;
                }
                while (__any_sync(0xffffffffu, (rem[0] | rem[1] | rem[2] | rem[3]) != 0u)) {
#pragma unroll
                    for (int u = 0; u < U4; u++) {
                        const int src = rem[u] ? __ffs(rem[u]) - 1 : lane;
#pragma unroll
                        for (int q = 0; q < NB; q++) {
                            const double x = __shfl_sync(0xffffffffu, v[u][q], src);
                            if (rem[u]) sum[u][q] += x;
                        }
                        rem[u] &= rem[u] - 1u;
                    }
                }
                // histogram updates in step order (a bin may recur in a later step, led by another lane)
#pragma unroll
                for (int u = 0; u < U4; u++) {
                    if (lead[u])
#pragma unroll
                        for (int q = 0; q < NB; q++) hist[bin[u] * NB + q] += sum[u][q];
                    __syncwarp();
                }
            }
        }
        if (TMA) __syncthreads();  // buffer j&1 is refilled by the copy issued in iteration j+1
    }
    __syncwarp();
    if (k < K)
        for (int a = lane; a < ns * NB; a += 32) P[((size_t)blockIdx.x * K + k) * ns * NB + a] = hist[a];
}

// U[(k*ns + l)*Bp + q] = sum over row ranges (fixed order) of P[range][k][l][q]; columns >= NB are 0
__global__ void k_narrow_combine(const double* __restrict__ P, int nranges, int K, int ns, int NB, int Bp,
                                 double* __restrict__ U) {
    const int64_t tot = (int64_t)K * ns * Bp;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int q = (int)(e % Bp);
        const int64_t g = e / Bp;  // k * ns + l
        double v = 0.0;
        if (q < NB)
            for (int c = 0; c < nranges; c++) v += P[((size_t)c * K * ns + g) * NB + q];
        U[e] = v;
    }
}

}  // namespace

// ===================================================================== host

static int ensure_ws(cwb_ctx* c, int32_t B, cudaStream_t s, bool need_rt = true) {
    cwb_train_ws& w = c->ws;
    const int Bp = (B + 31) / 32 * 32;
    const int nblk = (int)((c->n + kRowsH6 - 1) / kRowsH6);
    if (w.Bp >= Bp && w.B >= B && w.U && (w.Rt || !need_rt)) return CWB_OK;
    cwb_release(w.Rt, s); cwb_release(w.U, s); cwb_release(w.theta, s); cwb_release(w.delta, s);
    cwb_release(w.rr, s); cwb_release(w.zhat, s); cwb_release(w.kstar, s); cwb_release(w.part, s);
    cwb_release(w.narrow, s);
    cwb_release(w.colpart, s);
    cwb_release(w.acwb, s);
    cwb_release(w.pack, s);
    cwb_release(w.bern, s);
    cwb_release(w.fold, s);
    cwb_release(w.lbuf, s);
    w = cwb_train_ws();
    const size_t n = (size_t)c->n, K = c->K, ns = c->n_star, d = c->d;
    bool ok = true;
    if (need_rt) ok &= cwb_alloc((void**)&w.Rt, sizeof(double) * n * Bp, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&w.U, sizeof(double) * K * ns * Bp, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&w.theta, sizeof(double) * K * d * Bp, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&w.delta, sizeof(double) * K * Bp, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&w.rr, sizeof(double) * 2 * Bp, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&w.zhat, sizeof(double) * ns * Bp, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&w.kstar, sizeof(int32_t) * Bp, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&w.part, sizeof(double) * (size_t)nblk * Bp, s) == cudaSuccess;
    if (c->rows || c->nb) ok &= cwb_alloc((void**)&w.pack, sizeof(double) * (K * d + 1) * Bp, s) == cudaSuccess;
    if (!ok) return cwb_set_error(c, CWB_ENOMEM, "general-path workspace allocation failed");
    w.B = B; w.Bp = Bp; w.n_part = nblk;
    return CWB_OK;
}

template <typename PermT>
static void launch_h1(const double* Rt, int64_t n, int Bp, int K, int ns, const int32_t* off,
                      const void* perm, double* U, cudaStream_t s) {
    const int wpb = 8;
    dim3 grid((unsigned)(((int64_t)K * ns + wpb - 1) / wpb), Bp / 32);
    k_h1<PermT><<<grid, wpb * 32, 0, s>>>(Rt, n, Bp, K, ns, off, (const PermT*)perm, U);
}

// rows per chunk of the chunked H1: a 32-column tile of one chunk (rows x 256 B) well inside L2
static constexpr int64_t kH1ChunkBytes = 40ll << 20;  // R4 sweep: 24 MB 934, 40 MB 913, 64 MB 921, 96 MB 985 ms/step

#define H1W_LAUNCH(CH, GRID, OFF, CC, NCH, CHI)                                                            \
    do {                                                                                                   \
        if (perm_bytes == 2)                                                                               \
            k_h1w<uint16_t, CH><<<GRID, 256, 0, s>>>(Rt, n, Bp, K, ns, OFF, CC, NCH, CHI,                  \
                                                     (const uint16_t*)perm, U, tri_d);                     \
        else                                                                                               \
            k_h1w<uint32_t, CH><<<GRID, 256, 0, s>>>(Rt, n, Bp, K, ns, OFF, CC, NCH, CHI,                  \
                                                     (const uint32_t*)perm, U, tri_d);                     \
    } while (0)

// Row chunking of the general-path H1: when a column tile of the gathered matrix (n rows x tile_row bytes) exceeds
// L2, the bins are swept in row chunks of kH1ChunkBytes (per (learner, chunk, bin) row counts and starts, built
// once per pool and chunk size).  Returns the rows per chunk (0: one sweep) and sets *nch_out.
static int64_t h1_chunk_plan(cwb_ctx* c, int64_t tile_row, const int32_t* off, int K, int ns, int* nch_out,
                             cudaStream_t s) {
    const int64_t n = c->n;
    *nch_out = 1;
    if (!(n * tile_row > 80ll * 1000 * 1000 && c->h1_chunking && !c->rows && off == c->off)) return 0;
    static const int64_t chunk_bytes =
        getenv("CWB_H1_CHUNK_MB") ? (int64_t)atoi(getenv("CWB_H1_CHUNK_MB")) << 20 : kH1ChunkBytes;
    // equal chunks of at most chunk_bytes (R3: 3 x 66,667 rows = 34 MB instead of 2 x 81,920 + 36,160): the
    // measured sweep favours ~34 MB at R3 (profiles/r2h_h1_chunk.txt); the cached tables are keyed on the
    // rows per chunk
    const int64_t CR0 = std::max<int64_t>(1, chunk_bytes / tile_row);
    const int nch = (int)((n + CR0 - 1) / CR0);
    const int64_t CR = (n + nch - 1) / nch;
    if (!c->h1c || c->h1c_nch != nch || c->h1c_cr != CR) {  // per (learner, chunk, bin) counts / starts, once per pool
        cwb_release(c->h1c, s);
        c->h1c = nullptr;
        if (cwb_alloc((void**)&c->h1c, 2 * sizeof(uint32_t) * (size_t)K * nch * ns, s) != cudaSuccess) {
            cwb_set_error(c, CWB_ENOMEM, "chunked H1 tables");
            return -1;
        }
        c->h1c_nch = nch;
        c->h1c_cr = CR;
        k_h1_chunk_count<<<dim3(nch, K), 1024, sizeof(uint32_t) * ns, s>>>(c->idx, c->idx_bytes, n, ns, CR, nch,
                                                                         c->h1c);
        k_h1_chunk_start<<<(unsigned)(((int64_t)K * ns + 255) / 256), 256, 0, s>>>(c->h1c, c->off, K, ns, nch);
        c->launches += 2;
    }
    *nch_out = nch;
    return CR;
}

// one row chunk ch of the chunked H1 (U += the chunk's bin sums; chunk 0 writes)
static void h1_chunk(cwb_ctx* c, const double* Rt, int Bp, int K, int ns, const void* perm, int perm_bytes,
                     double* U, int nch, int ch, cudaStream_t s, int tri_d = 0) {
    const int64_t n = c->n;
    const int wpb = 8;
    dim3 grid((unsigned)(((int64_t)K * ns + wpb - 1) / wpb), Bp / 32);
    if (c->h1_wide && Bp % 64 == 0) {
        dim3 gw(grid.x, Bp / 64);
        H1W_LAUNCH(true, gw, nullptr, c->h1c, nch, ch);
    } else if (perm_bytes == 2) {
        k_h1c<uint16_t><<<grid, wpb * 32, 0, s>>>(Rt, n, Bp, K, ns, nch, ch, c->h1c, (const uint16_t*)perm, U);
    } else {
        k_h1c<uint32_t><<<grid, wpb * 32, 0, s>>>(Rt, n, Bp, K, ns, nch, ch, c->h1c, (const uint32_t*)perm, U);
    }
    c->launches++;
}

static void h1(cwb_ctx* c, const double* Rt, int Bp, int K, int ns, const int32_t* off,
               const void* perm, int perm_bytes, double* U, cudaStream_t s, int tri_d = 0) {
    const int64_t n = c->n;
    const bool wide = c->h1_wide && Bp % 64 == 0;
    const int64_t tile_row = wide ? 512 : 256;  // bytes of one row of the column tile a wave of warps gathers
    int nch = 1;
    const int64_t CR = h1_chunk_plan(c, tile_row, off, K, ns, &nch, s);
    if (CR < 0) return;
    if (CR > 0) {
        for (int ch = 0; ch < nch; ch++) h1_chunk(c, Rt, Bp, K, ns, perm, perm_bytes, U, nch, ch, s, tri_d);
        return;
    }
    if (wide && (int64_t)K * ns < INT32_MAX) {
        dim3 gw((unsigned)(((int64_t)K * ns + 7) / 8), Bp / 64);
        H1W_LAUNCH(false, gw, off, nullptr, 0, 0);
    } else if (perm_bytes == 2) {
        launch_h1<uint16_t>(Rt, n, Bp, K, ns, off, perm, U, s);
    } else {
        launch_h1<uint32_t>(Rt, n, Bp, K, ns, off, perm, U, s);
    }
    c->launches++;
}

// f0[b] = mean (center) and rr[b] = sum (y - f0)^2 of the B vectors Y[b][n] (I8)
static int column_stats(cwb_ctx* c, const double* Y, int B, bool center, double* f0, double* rr,
                        double* offset_out, cudaStream_t s, const uint8_t* mask = nullptr, int keep = 0,
                        const double* ncount = nullptr) {
    cwb_train_ws& w = c->ws;
    const int nblk = (int)((c->n + kColRows - 1) / kColRows);
    const size_t need = sizeof(double) * (size_t)nblk * B;
    if (w.colpart_bytes < need) {
        cwb_release(w.colpart, s);
        w.colpart = nullptr;
        w.colpart_bytes = 0;
        if (cwb_alloc((void**)&w.colpart, need, s) != cudaSuccess)
            return cwb_set_error(c, CWB_ENOMEM, "column statistics workspace allocation failed");
        w.colpart_bytes = need;
    }
    if (center) {
        k_colsum<<<dim3(nblk, B), 256, 0, s>>>(Y, c->n, nullptr, false, w.colpart, c->d_status, mask, keep);
        k_center_fin<<<(B + 127) / 128, 128, 0, s>>>(w.colpart, nblk, B, c->n, 0, f0, offset_out, ncount);
        c->launches += 2;
    }
    k_colsum<<<dim3(nblk, B), 256, 0, s>>>(Y, c->n, f0, true, w.colpart, c->d_status, mask, keep);
    k_center_fin<<<(B + 127) / 128, 128, 0, s>>>(w.colpart, nblk, B, c->n, 1, rr, nullptr);
    c->launches += 2;
    return CWB_OK;
}

// next (start, stop) event pair of the H1 timing hook, NULL when it is off
static cudaEvent_t* cwb_h1_events(cwb_ctx* c) {
    if (!c->h1_timing) return nullptr;
    if ((size_t)c->h1_ev_used + 2 > c->h1_ev.size()) {
        for (int i = 0; i < 64; i++) {
            cudaEvent_t e;
            if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
            c->h1_ev.push_back(e);
        }
    }
    cudaEvent_t* p = c->h1_ev.data() + c->h1_ev_used;
    c->h1_ev_used += 2;
    return p;
}

// one findBestBaselearner on the residual columns of ws.Rt
static void find_best_iter(cwb_ctx* c, int32_t B, double nu, int m, double* agg, int32_t* k_trace,
                           double* sse_trace, int32_t* k_out, double* theta_out, double* sse_out,
                           cudaStream_t s) {
    cwb_train_ws& w = c->ws;
    const int Bp = w.Bp;
    if (c->lshard) {  // learner sharding: H1-H4 on this rank's learners, one all-reduce of the candidates
        const int k0 = c->lk0, kl = c->lk1 - c->lk0, ns = c->n_star, d = c->d;
        const int world = c->world, rank = c->rank;
        const size_t cnt = (size_t)world * Bp * (d + 2);
        if (w.lbuf_bytes < cnt * sizeof(double)) {
            cwb_release(w.lbuf, s);
            w.lbuf = nullptr;
            w.lbuf_bytes = 0;
            if (cwb_alloc((void**)&w.lbuf, cnt * sizeof(double), s) != cudaSuccess) {
                cwb_set_error(c, CWB_ENOMEM, "learner-sharding buffer");
                return;
            }
            w.lbuf_bytes = cnt * sizeof(double);
        }
        const void* pk = (const char*)c->perm + (size_t)c->perm_bytes * k0 * c->n;
        if (c->perm_bytes == 2)
            launch_h1<uint16_t>(w.Rt, c->n, Bp, kl, ns, c->off + (size_t)k0 * (ns + 1), pk, w.U + (size_t)k0 * ns * Bp, s);
        else
            launch_h1<uint32_t>(w.Rt, c->n, Bp, kl, ns, c->off + (size_t)k0 * (ns + 1), pk, w.U + (size_t)k0 * ns * Bp, s);
        k_h234<<<dim3(kl, Bp / 32), 256, 0, s>>>(w.U + (size_t)k0 * ns * Bp, Bp, ns, d, c->ZT + (size_t)k0 * c->W * d,
                                                 c->W, c->lwin + (size_t)k0 * d * 2,
                                                 c->Ainv + (size_t)k0 * d * d, c->G + (size_t)k0 * d * d,
                                                 w.theta + (size_t)k0 * d * Bp, w.delta + (size_t)k0 * Bp);
        cudaMemsetAsync(w.lbuf, 0, cnt * sizeof(double), s);
        k_lshard_pack<<<(B + 127) / 128, 128, 0, s>>>(w.delta, w.theta, k0, k0 + kl, d, B, Bp, rank, w.lbuf);
        c->launches += 3;
        if (cwb_rows_allreduce(c, w.lbuf, (int64_t)cnt, s)) return;
        k_lshard_pick<<<(Bp + 127) / 128, 128, 0, s>>>(w.lbuf, world, w.rr, c->K, d, B, Bp, nu, m, w.kstar, w.theta,
                                                       agg, k_trace, sse_trace, k_out, theta_out, sse_out);
        c->launches += 1;
        return;
    }
    if (c->nb) {  // unbinned learners: s = Z^T r by the 4-tap scatter (cwb_nb.cu), then H3-H4 from s
        cwb_nb_h12(c, w.Rt, Bp, w.pack, s);
        k_h234<<<dim3(c->K, Bp / 32), 256, 0, s>>>(w.U, Bp, c->n_star, c->d, c->ZT, c->W, c->lwin, c->Ainv,
                                                    c->G, w.theta, w.delta, nullptr, nullptr, nullptr, 0, w.pack, 2);
    } else {
        cudaEvent_t* ev = cwb_h1_events(c);  // profiling hook (bench.py's roofline): H1 bracketed by events
        if (ev) cudaEventRecord(ev[0], s);
        h1(c, w.Rt, Bp, c->K, c->n_star, c->off, c->perm, c->perm_bytes, w.U, s);
        if (ev) cudaEventRecord(ev[1], s);
        k_h234<<<dim3(c->K, Bp / 32), 256, 0, s>>>(w.U, Bp, c->n_star, c->d, c->ZT, c->W, c->lwin,
                                                    c->Ainv, c->G, w.theta, w.delta);
    }
    k_h5<<<Bp / 32, 256, 0, s>>>(w.delta, w.theta, w.rr, c->K, c->d, B, Bp, nu, m, w.kstar,
                                          agg, k_trace, sse_trace, k_out, theta_out, sse_out);
    c->launches += 2;
}

template <typename IdxT, int NB>
static void launch_narrow(bool tma, const double* R, int64_t n, int K, int ns, const void* idx, int64_t rpc, int nc,
                          int nranges, int groups, size_t smem, double* P, cudaStream_t s) {
    if (tma) {
        auto kern = k_h1_narrow<IdxT, NB, true>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<dim3(nranges, groups), 256, smem, s>>>(R, n, K, ns, (const IdxT*)idx, rpc, nc, P);
    } else {
        auto kern = k_h1_narrow<IdxT, NB, false>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<dim3(nranges, groups), 256, smem, s>>>(R, n, K, ns, (const IdxT*)idx, rpc, nc, P);
    }
}

// findBestBaselearner for B <= 4 residual vectors: narrow H1 + combine, then the general H2-H5
static int find_best_narrow(cwb_ctx* c, const double* R, int32_t B, int32_t* k_out, double* theta_out,
                            double* sse_out, cudaStream_t s) {
    int rc = ensure_ws(c, B, s, false);
    if (rc) return rc;
    cwb_train_ws& w = c->ws;
    const int K = c->K, ns = c->n_star, LPC = 8, groups = (K + LPC - 1) / LPC;
    const size_t hist = sizeof(double) * (size_t)LPC * ns * B;
    const size_t per_row = sizeof(double) * B + (size_t)c->idx_bytes * LPC;  // staged bytes per chunk row
    // TMA bulk copies need 16-byte aligned chunk starts: n a multiple of 16 rows, R 16-byte aligned
    const bool tma = (c->n % 16) == 0 && ((uintptr_t)R & 15) == 0;
    const int nbuf = tma ? 2 : 1;
    if (hist + nbuf * per_row * 512 > 200 * 1024) return CWB_EUNSUPPORTED;
    int nc = 16384;  // rows staged per chunk, within ~110 KB (two CTAs per SM) if possible
    while (nc > 512 && hist + nbuf * per_row * nc > 110 * 1024) nc >>= 1;
    while (nc > 512 && hist + nbuf * per_row * nc > 200 * 1024) nc >>= 1;
    int nranges = (int)std::max<int64_t>(1, std::min<int64_t>((2 * cwb_num_sms() + groups - 1) / groups, (c->n + nc - 1) / nc));
    const int64_t rpc = ((c->n + nranges - 1) / nranges + 15) / 16 * 16;  // 16-row aligned range starts
    nranges = (int)((c->n + rpc - 1) / rpc);
    const size_t need = sizeof(double) * (size_t)nranges * K * ns * B;
    if (w.narrow_bytes < need) {
        cwb_release(w.narrow, s);
        w.narrow = nullptr;
        w.narrow_bytes = 0;
        if (cwb_alloc((void**)&w.narrow, need, s) != cudaSuccess)
            return cwb_set_error(c, CWB_ENOMEM, "narrow find_best workspace allocation failed");
        w.narrow_bytes = need;
    }
    const size_t smem = hist + nbuf * per_row * nc;
    rc = column_stats(c, R, B, false, nullptr, w.rr, nullptr, s);
    if (rc) return rc;
    // streaming gather plan (cwb_stream.cu) when it applies, else the MATCH.ANY histograms
#define NARROW_CASE(IT)                                                                                          \
    switch (B) {                                                                                                 \
        case 1: launch_narrow<IT, 1>(tma, R, c->n, K, ns, c->idx, rpc, nc, nranges, groups, smem, w.narrow, s); break; \
        case 2: launch_narrow<IT, 2>(tma, R, c->n, K, ns, c->idx, rpc, nc, nranges, groups, smem, w.narrow, s); break; \
        case 3: launch_narrow<IT, 3>(tma, R, c->n, K, ns, c->idx, rpc, nc, nranges, groups, smem, w.narrow, s); break; \
        default: launch_narrow<IT, 4>(tma, R, c->n, K, ns, c->idx, rpc, nc, nranges, groups, smem, w.narrow, s); break; \
    }
    {
        if (c->idx_bytes == 1) NARROW_CASE(uint8_t) else NARROW_CASE(uint16_t)
#undef NARROW_CASE
        const int64_t tot = (int64_t)K * ns * w.Bp;
        k_narrow_combine<<<(unsigned)std::min<int64_t>(4 * 1184, (tot + 255) / 256), 256, 0, s>>>(
            w.narrow, nranges, K, ns, B, w.Bp, w.U);
        c->launches += 2;
    }
    k_h234<<<dim3(K, w.Bp / 32), 256, 0, s>>>(w.U, w.Bp, ns, c->d, c->ZT, c->W, c->lwin, c->Ainv, c->G, w.theta,
                                              w.delta);
    k_h5<<<w.Bp / 32, 256, 0, s>>>(w.delta, w.theta, w.rr, K, c->d, B, w.Bp, 0.0, 0, w.kstar, nullptr,
                                            nullptr, nullptr, k_out, theta_out, sse_out);
    c->launches += 2;
    return cwb_check_launch(c, "narrow find_best kernels");
}

int cwb_find_best_general(cwb_ctx* c, const double* R, int32_t B, int32_t* k_out, double* theta_out,
                          double* sse_out, cudaStream_t s) {
    if (B <= 4 && c->path != 2 && c->narrow_mode == 0) {
        const int rc = cwb_find_best_stream(c, R, B, k_out, theta_out, sse_out, s);
        if (rc != CWB_EUNSUPPORTED) return rc;
    }
    if (B <= 4 && c->path != 2) {
        const int rc = find_best_narrow(c, R, B, k_out, theta_out, sse_out, s);
        if (rc != CWB_EUNSUPPORTED) return rc;
    }
    int rc = ensure_ws(c, B, s);
    if (rc) return rc;
    cwb_train_ws& w = c->ws;
    rc = column_stats(c, R, B, false, nullptr, w.rr, nullptr, s);
    if (rc) return rc;
    dim3 gt((unsigned)((c->n + 31) / 32), w.Bp / 32);
    k_tr_in<<<gt, dim3(32, 8), 0, s>>>(R, c->n, B, w.Bp, nullptr, nullptr, w.Rt);
    c->launches += 1;
    find_best_iter(c, B, 0.0, 0, nullptr, nullptr, nullptr, k_out, theta_out, sse_out, s);
    if (c->status) return c->status;
    return cwb_check_launch(c, "find_best kernels");
}

// H6 launch: k_h6s when a block's zhat columns fit in shared memory (CB = 32, else 16), else k_h6.  The grid
// has X row blocks per column block with X * (Bp / CB) a multiple of the SM count (whole waves of one block per
// SM).  Returns the number of row-block partials written to part (k_rr's nblk).  CWB_H6=0 forces k_h6 (A/B).
template <typename IdxT>
static int launch_h6_t(cwb_ctx* c, double* Rt, int Bp, const int32_t* kstar, const double* zhat, double* part,
                       int nblk_max, cudaStream_t s) {
    static const int mode = getenv("CWB_H6") ? atoi(getenv("CWB_H6")) : 1;
    const int ns = c->n_star;
    int cb = 0;
    if (mode && (size_t)ns * 32 * sizeof(double) <= 160 * 1024) cb = 32;
    else if (mode && (size_t)ns * 16 * sizeof(double) <= 160 * 1024) cb = 16;
    if (cb) {
        const int Y = Bp / cb, nsm = cwb_num_sms();
        const int X = std::max(1, std::min(nblk_max, nsm / std::gcd(nsm, Y)));
        const int64_t rpb = (c->n + X - 1) / X;
        const size_t smem = sizeof(double) * (size_t)ns * cb;
        if (cb == 32) {
            static bool attr = false;
            if (!attr) { cudaFuncSetAttribute(k_h6s<IdxT, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024); attr = true; }
            k_h6s<IdxT, 32><<<dim3(X, Y), kH6sThreads, smem, s>>>(Rt, c->n, Bp, kstar, (const IdxT*)c->idx, zhat, ns,
                                                                 rpb, part);
        } else {
            static bool attr = false;
            if (!attr) { cudaFuncSetAttribute(k_h6s<IdxT, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024); attr = true; }
            k_h6s<IdxT, 16><<<dim3(X, Y), kH6sThreads, smem, s>>>(Rt, c->n, Bp, kstar, (const IdxT*)c->idx, zhat, ns,
                                                                 rpb, part);
        }
        return X;
    }
    k_h6<IdxT><<<dim3(nblk_max, Bp / 32), 256, 0, s>>>(Rt, c->n, Bp, kstar, (const IdxT*)c->idx, zhat, part);
    return nblk_max;
}
static int launch_h6(cwb_ctx* c, double* Rt, int Bp, const int32_t* kstar, const double* zhat, double* part,
                     int nblk_max, cudaStream_t s) {
    return c->idx_bytes == 1 ? launch_h6_t<uint8_t>(c, Rt, Bp, kstar, zhat, part, nblk_max, s)
                             : launch_h6_t<uint16_t>(c, Rt, Bp, kstar, zhat, part, nblk_max, s);
}

int cwb_train_general(cwb_ctx* c, const double* Y, int32_t B, double nu, int32_t M,
                      double* offset_out, double* theta_agg_out, int32_t* k_trace,
                      double* sse_trace, double* risk_trace, cudaStream_t s) {
    int rc = ensure_ws(c, B, s);
    if (rc) return rc;
    cwb_train_ws& w = c->ws;
    const int Bp = w.Bp;
    double* off_ws = w.rr + Bp;
    rc = column_stats(c, Y, B, true, off_ws, w.rr, offset_out, s);
    if (rc) return rc;
    dim3 gt((unsigned)((c->n + 31) / 32), Bp / 32);
    k_tr_in<<<gt, dim3(32, 8), 0, s>>>(Y, c->n, B, Bp, off_ws, nullptr, w.Rt);
    const size_t nagg = (size_t)B * c->K * c->d;
    k_zero<<<(unsigned)min((size_t)1184, (nagg + 255) / 256 + 1), 256, 0, s>>>(theta_agg_out, nagg);
    c->launches += 3;
    const int nblk = w.n_part;
    for (int m = 0; m < M; m++) {
        find_best_iter(c, B, nu, m, theta_agg_out, k_trace, sse_trace, nullptr, nullptr, nullptr, s);
        if (c->nb) {
            cwb_nb_h6(c, w.Rt, Bp, w.kstar, w.theta, nu, kRowsH6, nblk, w.part, s);
            k_rr<<<Bp / 32, kRrThreads, 0, s>>>(w.part, nblk, B, Bp, c->n, m, w.rr, risk_trace);
            c->launches += 1;
            continue;
        }
        k_zhat<<<dim3((c->n_star + 7) / 8, Bp / 32), 256, 0, s>>>(w.kstar, w.theta, c->zj0, c->Zs,
                                                                  c->n_star, c->d, B, Bp, nu, B, nu, w.zhat);
        const int nb6 = launch_h6(c, w.Rt, Bp, w.kstar, w.zhat, w.part, nblk, s);
        k_rr<<<Bp / 32, kRrThreads, 0, s>>>(w.part, nb6, B, Bp, c->n, m, w.rr, risk_trace);
        c->launches += 3;
        if (c->status) return c->status;  // e.g. a failed collective of learner sharding
    }
    return cwb_check_launch(c, "general train kernels");
}

// CWB with the Bernoulli loss on the general path (kernels above).
int cwb_train_bernoulli_general(cwb_ctx* c, const double* Y, int32_t B, double nu, int32_t M,
                                double* offset_out, double* theta_agg_out, int32_t* k_trace,
                                double* sse_trace, double* risk_trace, cudaStream_t s) {
    int rc = ensure_ws(c, B, s);
    if (rc) return rc;
    cwb_train_ws& w = c->ws;
    const int Bp = w.Bp;
    const int nblk = w.n_part;
    const size_t need = sizeof(double) * ((size_t)2 * c->n * Bp + (size_t)2 * nblk * Bp);
    if (w.bern_bytes < need) {
        cwb_release(w.bern, s);
        w.bern = nullptr;
        w.bern_bytes = 0;
        if (cwb_alloc((void**)&w.bern, need, s) != cudaSuccess)
            return cwb_set_error(c, CWB_ENOMEM, "Bernoulli workspace allocation failed");
        w.bern_bytes = need;
    }
    double* F = w.bern;
    double* Yt = F + (size_t)c->n * Bp;
    double* part = Yt + (size_t)c->n * Bp;
    double* f0 = w.rr + Bp;
    rc = column_stats(c, Y, B, true, f0, w.rr, nullptr, s);  // f0 = mean(y), finiteness
    if (rc) return rc;
    dim3 gt((unsigned)((c->n + 31) / 32), Bp / 32);
    k_bern_init<<<gt, dim3(32, 8), 0, s>>>(Y, c->n, B, Bp, Yt, c->d_status);
    k_bern_offset<<<(B + 127) / 128, 128, 0, s>>>(f0, B, offset_out, c->d_status);
    const size_t nagg = (size_t)B * c->K * c->d;
    k_zero<<<(unsigned)min((size_t)1184, (nagg + 255) / 256 + 1), 256, 0, s>>>(theta_agg_out, nagg);
    dim3 g6(nblk, Bp / 32);
    auto update = [&](bool first) {
        if (c->idx_bytes == 1)
            k_bern_update<uint8_t><<<g6, 256, 0, s>>>(w.Rt, F, Yt, c->n, Bp, B, first ? f0 : nullptr, w.kstar,
                                                      (const uint8_t*)c->idx, first ? nullptr : w.zhat, part, nblk);
        else
            k_bern_update<uint16_t><<<g6, 256, 0, s>>>(w.Rt, F, Yt, c->n, Bp, B, first ? f0 : nullptr, w.kstar,
                                                       (const uint16_t*)c->idx, first ? nullptr : w.zhat, part, nblk);
    };
    update(true);  // f = f0, r = y - sigma(f0), r^T r
    k_bern_rr<<<(B + 127) / 128, 128, 0, s>>>(part, nblk, B, Bp, c->n, -1, w.rr, nullptr);
    c->launches += 5;
    for (int m = 0; m < M; m++) {
        find_best_iter(c, B, nu, m, theta_agg_out, k_trace, sse_trace, nullptr, nullptr, nullptr, s);
        k_zhat<<<dim3((c->n_star + 7) / 8, Bp / 32), 256, 0, s>>>(w.kstar, w.theta, c->zj0, c->Zs,
                                                                  c->n_star, c->d, B, Bp, nu, B, nu, w.zhat);
        update(false);
        k_bern_rr<<<(B + 127) / 128, 128, 0, s>>>(part, nblk, B, Bp, c->n, m, w.rr, risk_trace);
        c->launches += 3;
    }
    return cwb_check_launch(c, "Bernoulli train kernels");
}

// CWB with per-replication CV folds on the general path (kernels above).
int cwb_train_folds_general(cwb_ctx* c, const double* Y, int32_t B, const uint8_t* fold_of_row, int32_t F,
                            const int32_t* fold_of_rep, double nu, int32_t M, double* offset_out,
                            double* theta_agg_out, int32_t* k_trace, double* sse_trace, double* risk_trace,
                            double* val_risk_trace, cudaStream_t s) {
    int rc = ensure_ws(c, B, s);
    if (rc) return rc;
    cwb_train_ws& w = c->ws;
    const int Bp = w.Bp, K = c->K, ns = c->n_star, d = c->d;
    const int nblk = w.n_part;
    // per fold: G_f, A_f^-1 (K x d x d each); per column: f0, training / held-out counts;
    // partials 2 x nblk x Bp; column folds (padded); training-row bin counts; a fold mask (n bytes)
    const size_t dbl = 2 * (size_t)F * K * d * d + 3 * (size_t)Bp + 2 * (size_t)nblk * Bp;
    const size_t need = sizeof(double) * dbl + sizeof(int32_t) * Bp + sizeof(uint32_t) * (size_t)K * ns +
                        (size_t)c->n + 16;
    if (w.fold_bytes < need) {
        cwb_release(w.fold, s);
        w.fold = nullptr;
        w.fold_bytes = 0;
        if (cwb_alloc((void**)&w.fold, need, s) != cudaSuccess)
            return cwb_set_error(c, CWB_ENOMEM, "CV-fold workspace allocation failed");
        w.fold_bytes = need;
    }
    double* Gs = w.fold;
    double* As = Gs + (size_t)F * K * d * d;
    double* f0 = As + (size_t)F * K * d * d;
    double* ntr = f0 + Bp;
    double* nho = ntr + Bp;
    double* part = nho + Bp;
    int32_t* colfold = (int32_t*)(part + 2 * (size_t)nblk * Bp);
    uint32_t* cnt_tr = (uint32_t*)(colfold + Bp);
    uint8_t* mask = (uint8_t*)(cnt_tr + (size_t)K * ns);
    k_fill_int<<<(Bp + 127) / 128, 128, 0, s>>>(colfold, Bp, -1);
    CWB_CUDA_TRY(c, cudaMemcpyAsync(colfold, fold_of_rep, sizeof(int32_t) * B, cudaMemcpyDeviceToDevice, s));
    // argument checks first (a replication without training rows is CWB_EINVAL, not a singular table)
    k_fold_stats<<<B, 256, 0, s>>>(Y, c->n, fold_of_row, F, colfold, f0, w.rr, ntr, nho, offset_out, c->d_status);
    const int gx = (int)std::min<int64_t>(1184, (c->n + 255) / 256);
    for (int f = 0; f < F; f++) {  // training-row tables of fold f (binMatMat with 0/1 weights)
        k_fold_mask<<<gx, 256, 0, s>>>(fold_of_row, c->n, f, mask);
        rc = cwb_launch_masked_pool(c, mask, cnt_tr, Gs + (size_t)f * K * d * d, As + (size_t)f * K * d * d, s);
        if (rc) return rc;
        c->launches += 1;
    }
    dim3 gt((unsigned)((c->n + 31) / 32), Bp / 32);
    k_tr_in<<<gt, dim3(32, 8), 0, s>>>(Y, c->n, B, Bp, f0, nullptr, w.Rt);
    const size_t nagg = (size_t)B * K * d;
    k_zero<<<(unsigned)min((size_t)1184, (nagg + 255) / 256 + 1), 256, 0, s>>>(theta_agg_out, nagg);
    c->launches += 4;
    for (int m = 0; m < M; m++) {
        const int wpb = 8;
        dim3 grid((unsigned)(((int64_t)K * ns + wpb - 1) / wpb), Bp / 32);
        if (c->perm_bytes == 2)
            k_h1<uint16_t><<<grid, wpb * 32, 0, s>>>(w.Rt, c->n, Bp, K, ns, c->off, (const uint16_t*)c->perm, w.U,
                                                    fold_of_row, colfold);
        else
            k_h1<uint32_t><<<grid, wpb * 32, 0, s>>>(w.Rt, c->n, Bp, K, ns, c->off, (const uint32_t*)c->perm, w.U,
                                                    fold_of_row, colfold);
        k_h234<<<dim3(K, Bp / 32), 256, 0, s>>>(w.U, Bp, ns, d, c->ZT, c->W, c->lwin, c->Ainv, c->G, w.theta,
                                                w.delta, nullptr, nullptr, nullptr, 0, nullptr, 0, As, Gs, colfold);
        k_h5<<<Bp / 32, 256, 0, s>>>(w.delta, w.theta, w.rr, K, d, B, Bp, nu, m, w.kstar, theta_agg_out,
                                              k_trace, sse_trace, nullptr, nullptr, nullptr);
        k_zhat<<<dim3((ns + 7) / 8, Bp / 32), 256, 0, s>>>(w.kstar, w.theta, c->zj0, c->Zs, ns, d, B, Bp, nu, B, nu,
                                                           w.zhat);
        dim3 g6(nblk, Bp / 32);
        if (c->idx_bytes == 1)
            k_h6_fold<uint8_t><<<g6, 256, 0, s>>>(w.Rt, c->n, Bp, w.kstar, (const uint8_t*)c->idx, w.zhat, fold_of_row,
                                                  colfold, B, part, nblk);
        else
            k_h6_fold<uint16_t><<<g6, 256, 0, s>>>(w.Rt, c->n, Bp, w.kstar, (const uint16_t*)c->idx, w.zhat,
                                                   fold_of_row, colfold, B, part, nblk);
        k_rr_fold<<<(B + 127) / 128, 128, 0, s>>>(part, nblk, B, Bp, ntr, nho, m, w.rr, risk_trace, val_risk_trace);
        c->launches += 6;
    }
    return cwb_check_launch(c, "CV-fold train kernels");
}

// ------------------------------------------------------------ row sharding
// include/cwb.h "row sharding": the context holds rows [row0, row0 + n) of n_glob.
// Per iteration: local H1 and s = Zb^T u (k_h234 smode 1) into pack[K][d][Bp], the local
// r^T r in pack[K d Bp ..]; one all-reduce of the pack; then H3-H5 from the summed s and
// r^T r on every rank (identical bytes in -> identical k*, theta), H6 on the local rows.

// column sums of Y[B][n] (local rows) into out[B]: sum y (f0 == nullptr, sq false) or sum (y - f0)^2
static int col_sums(cwb_ctx* c, const double* Y, int B, const double* f0, bool sq, double* out, cudaStream_t s) {
    cwb_train_ws& w = c->ws;
    const int nblk = (int)((c->n + kColRows - 1) / kColRows);
    const size_t need = sizeof(double) * (size_t)nblk * B;
    if (w.colpart_bytes < need) {
        cwb_release(w.colpart, s);
        w.colpart = nullptr;
        w.colpart_bytes = 0;
        if (cwb_alloc((void**)&w.colpart, need, s) != cudaSuccess)
            return cwb_set_error(c, CWB_ENOMEM, "column statistics workspace allocation failed");
        w.colpart_bytes = need;
    }
    k_colsum<<<dim3(nblk, B), 256, 0, s>>>(Y, c->n, f0, sq, w.colpart, c->d_status);
    k_center_fin<<<(B + 127) / 128, 128, 0, s>>>(w.colpart, nblk, B, c->n, 1, out, nullptr);
    c->launches += 2;
    return CWB_OK;
}

// H1 + s on the local rows, all-reduce of (s, r^T r), H3-H5 (k_h5 reads the summed r^T r)
static int find_best_rows_iter(cwb_ctx* c, int32_t B, double nu, int m, double* agg, int32_t* k_trace,
                               double* sse_trace, int32_t* k_out, double* theta_out, double* sse_out,
                               double* risk_prev, cudaStream_t s) {
    cwb_train_ws& w = c->ws;
    const int Bp = w.Bp, K = c->K, d = c->d;
    double* rr_g = w.pack + (size_t)K * d * Bp;
    h1(c, w.Rt, Bp, K, c->n_star, c->off, c->perm, c->perm_bytes, w.U, s);
    k_h234<<<dim3(K, Bp / 32), 256, 0, s>>>(w.U, Bp, c->n_star, d, c->ZT, c->W, c->lwin, c->Ainv, c->G, w.theta,
                                            w.delta, nullptr, nullptr, nullptr, 0, w.pack, 1);
    c->launches += 1;
    int rc = cwb_check_launch(c, "row-sharded s kernels");
    if (rc) return rc;
    rc = cwb_rows_allreduce(c, w.pack, (int64_t)(K * d + 1) * Bp, s);
    if (rc) return rc;
    if (risk_prev) {
        k_risk<<<(B + 127) / 128, 128, 0, s>>>(rr_g, B, c->n_glob, risk_prev);
        c->launches += 1;
    }
    k_h234<<<dim3(K, Bp / 32), 256, 0, s>>>(w.U, Bp, c->n_star, d, c->ZT, c->W, c->lwin, c->Ainv, c->G, w.theta,
                                            w.delta, nullptr, nullptr, nullptr, 0, w.pack, 2);
    k_h5<<<Bp / 32, 256, 0, s>>>(w.delta, w.theta, rr_g, K, d, B, Bp, nu, m, w.kstar, agg, k_trace,
                                          sse_trace, k_out, theta_out, sse_out);
    c->launches += 2;
    return CWB_OK;
}

int cwb_find_best_rows(cwb_ctx* c, const double* R, int32_t B, int32_t* k_out, double* theta_out,
                       double* sse_out, cudaStream_t s) {
    int rc = ensure_ws(c, B, s);
    if (rc) return rc;
    cwb_train_ws& w = c->ws;
    const int Bp = w.Bp;
    double* rr_g = w.pack + (size_t)c->K * c->d * Bp;
    CWB_CUDA_TRY(c, cudaMemsetAsync(rr_g, 0, sizeof(double) * Bp, s));
    rc = col_sums(c, R, B, nullptr, true, rr_g, s);  // local r^T r (f0 = 0)
    if (rc) return rc;
    dim3 gt((unsigned)((c->n + 31) / 32), Bp / 32);
    k_tr_in<<<gt, dim3(32, 8), 0, s>>>(R, c->n, B, Bp, nullptr, nullptr, w.Rt);
    c->launches += 1;
    rc = find_best_rows_iter(c, B, 0.0, 0, nullptr, nullptr, nullptr, k_out, theta_out, sse_out, nullptr, s);
    if (rc) return rc;
    return cwb_check_launch(c, "row-sharded find_best kernels");
}

int cwb_train_rows(cwb_ctx* c, const double* Y, int32_t B, double nu, int32_t M, double* offset_out,
                   double* theta_agg_out, int32_t* k_trace, double* sse_trace, double* risk_trace, cudaStream_t s) {
    int rc = ensure_ws(c, B, s);
    if (rc) return rc;
    cwb_train_ws& w = c->ws;
    const int Bp = w.Bp;
    double* rr_g = w.pack + (size_t)c->K * c->d * Bp;
    double* f0 = w.rr + Bp;
    CWB_CUDA_TRY(c, cudaMemsetAsync(rr_g, 0, sizeof(double) * Bp, s));
    // f0 = mean over all rows: local sums, all-reduce, / n_glob
    rc = col_sums(c, Y, B, nullptr, false, rr_g, s);
    if (rc) return rc;
    rc = cwb_rows_allreduce(c, rr_g, Bp, s);
    if (rc) return rc;
    k_mean_glob<<<(B + 127) / 128, 128, 0, s>>>(rr_g, B, c->n_glob, f0, offset_out);
    c->launches += 1;
    rc = col_sums(c, Y, B, f0, true, rr_g, s);  // local r^T r, summed by the first iteration's all-reduce
    if (rc) return rc;
    dim3 gt((unsigned)((c->n + 31) / 32), Bp / 32);
    k_tr_in<<<gt, dim3(32, 8), 0, s>>>(Y, c->n, B, Bp, f0, nullptr, w.Rt);
    const size_t nagg = (size_t)B * c->K * c->d;
    k_zero<<<(unsigned)min((size_t)1184, (nagg + 255) / 256 + 1), 256, 0, s>>>(theta_agg_out, nagg);
    c->launches += 2;
    const int nblk = w.n_part;
    for (int m = 0; m < M; m++) {
        double* risk_prev = (risk_trace && m > 0) ? risk_trace + (size_t)(m - 1) * B : nullptr;
        rc = find_best_rows_iter(c, B, nu, m, theta_agg_out, k_trace, sse_trace, nullptr, nullptr, nullptr,
                                 risk_prev, s);
        if (rc) return rc;
        k_zhat<<<dim3((c->n_star + 7) / 8, Bp / 32), 256, 0, s>>>(w.kstar, w.theta, c->zj0, c->Zs, c->n_star,
                                                                  c->d, B, Bp, nu, B, nu, w.zhat);
        const int nb6 = launch_h6(c, w.Rt, Bp, w.kstar, w.zhat, w.part, nblk, s);
        k_rr<<<Bp / 32, kRrThreads, 0, s>>>(w.part, nb6, B, Bp, c->n, m, rr_g, nullptr);  // local r^T r
        c->launches += 3;
    }
    if (M > 0 && risk_trace) {  // the last iteration's risk needs one more sum
        rc = cwb_rows_allreduce(c, rr_g, Bp, s);
        if (rc) return rc;
        k_risk<<<(B + 127) / 128, 128, 0, s>>>(rr_g, B, c->n_glob, risk_trace + (size_t)(M - 1) * B);
        c->launches += 1;
    }
    return cwb_check_launch(c, "row-sharded train kernels");
}

// ------------------------------------------------ stand-alone primitives
namespace {
__global__ void k_gram_dense(const double* __restrict__ Zb, const double* __restrict__ u, int ustride,
                             int ns, int d, double* __restrict__ out) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < d * d; e += gridDim.x * blockDim.x) {
        const int a = e / d, b = e % d;
        double s = 0.0;
        for (int l = 0; l < ns; l++) s += u[(size_t)l * ustride] * (Zb[(size_t)l * d + a] * Zb[(size_t)l * d + b]);
        out[e] = s;
    }
}
__global__ void k_fill(double* p, int64_t cnt, double v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}
}  // namespace

// caller-supplied index vectors of the standalone binMatVec / binMatMat calls: every idx(i) < n* (ADVICE r1:
// the bin inversion would otherwise count and scatter outside its arrays)
template <typename IdxT>
__global__ void k_idx_check(const IdxT* __restrict__ idx, int64_t n, int ns, int* bad) {
    int b = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        b |= (int)idx[i] >= ns;
    if (__syncthreads_or(b) && threadIdx.x == 0) *bad = 1;
}

// U[l][b] = sum_{i: idx(i) = l} w_i R[b][i]  (binMatVec's u), rows in increasing order
static int binned_sums(const void* idx, int32_t idx_bytes, const double* w, const double* R, int64_t n,
                       int32_t B, int32_t ns, double* U, int Bp, cudaStream_t s) {
    const int perm_bytes = n <= 65536 ? 2 : 4;
    uint32_t* cnt = nullptr;
    int32_t* off = nullptr;
    void* perm = nullptr;
    double* Rt = nullptr;
    bool ok = cwb_alloc((void**)&cnt, sizeof(uint32_t) * ns, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&off, sizeof(int32_t) * (ns + 1), s) == cudaSuccess;
    ok &= cwb_alloc(&perm, (size_t)perm_bytes * n, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&Rt, sizeof(double) * (size_t)n * Bp, s) == cudaSuccess;
    int rc = ok ? CWB_OK : CWB_ENOMEM;
    if (rc == CWB_OK) {  // validate the index vector (one flag, read back: these are stand-alone calls)
        int* bad = reinterpret_cast<int*>(cnt);
        int hbad = 0;
        cudaMemsetAsync(bad, 0, sizeof(int), s);
        const unsigned g = (unsigned)std::min<int64_t>(1184, (n + 255) / 256);
        if (idx_bytes == 1) k_idx_check<uint8_t><<<g, 256, 0, s>>>((const uint8_t*)idx, n, ns, bad);
        else k_idx_check<uint16_t><<<g, 256, 0, s>>>((const uint16_t*)idx, n, ns, bad);
        if (cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess) rc = CWB_ECUDA;
        else if (hbad) rc = CWB_EINVAL;
    }
    if (rc == CWB_OK) rc = cwb_launch_csr(nullptr, idx, idx_bytes, n, 1, ns, cnt, off, perm, perm_bytes, s);
    if (rc == CWB_OK) {
        dim3 gt((unsigned)((n + 31) / 32), Bp / 32);
        k_tr_in<<<gt, dim3(32, 8), 0, s>>>(R, n, B, Bp, nullptr, w, Rt);
        const int wpb = 8;
        dim3 grid((unsigned)((ns + wpb - 1) / wpb), Bp / 32);
        if (perm_bytes == 2) k_h1<uint16_t><<<grid, 256, 0, s>>>(Rt, n, Bp, 1, ns, off, (const uint16_t*)perm, U);
        else k_h1<uint32_t><<<grid, 256, 0, s>>>(Rt, n, Bp, 1, ns, off, (const uint32_t*)perm, U);
        if (cudaGetLastError() != cudaSuccess) rc = CWB_ECUDA;
    }
    cwb_release(cnt, s); cwb_release(off, s); cwb_release(perm, s); cwb_release(Rt, s);
    return rc;
}

int cwb_bin_mat_vec_impl(const double* Zb, int32_t ns, int32_t d, const void* idx, int32_t idx_bytes,
                         const double* w, const double* R, int64_t n, int32_t B, double* out,
                         cudaStream_t s) {
    const int Bp = (B + 31) / 32 * 32;
    double* U = nullptr;
    if (cwb_alloc((void**)&U, sizeof(double) * (size_t)ns * Bp, s) != cudaSuccess) return CWB_ENOMEM;
    int rc = binned_sums(idx, idx_bytes, w, R, n, B, ns, U, Bp, s);
    if (rc == CWB_OK) {
        k_dense_proj<<<dim3((d + 7) / 8, Bp / 32), 256, 0, s>>>(Zb, U, ns, d, B, Bp, out);
        if (cudaGetLastError() != cudaSuccess) rc = CWB_ECUDA;
    }
    cwb_release(U, s);
    return rc;
}

// binMatMat: c_l = sum_{i in bin l} w_i, out = Zb^T diag(c) Zb
int cwb_bin_mat_mat_impl(const double* Zb, int32_t ns, int32_t d, const void* idx, int32_t idx_bytes,
                         const double* w, int64_t n, double* out, cudaStream_t s) {
    double *ones = nullptr, *U = nullptr;
    bool ok = cwb_alloc((void**)&U, sizeof(double) * (size_t)ns * 32, s) == cudaSuccess;
    if (!w) {
        ok &= cwb_alloc((void**)&ones, sizeof(double) * (size_t)n, s) == cudaSuccess;
        if (ok) k_fill<<<(unsigned)min((int64_t)1184, (n + 255) / 256), 256, 0, s>>>(ones, n, 1.0);
    }
    int rc = ok ? CWB_OK : CWB_ENOMEM;
    if (rc == CWB_OK) rc = binned_sums(idx, idx_bytes, nullptr, w ? w : ones, n, 1, ns, U, 32, s);
    if (rc == CWB_OK) {
        // U is ns x 32 with the sums in column 0 (stride 32)
        k_gram_dense<<<(d * d + 255) / 256, 256, 0, s>>>(Zb, U, 32, ns, d, out);
        if (cudaGetLastError() != cudaSuccess) rc = CWB_ECUDA;
    }
    cwb_release(ones, s);
    cwb_release(U, s);
    return rc;
}

// ===================================================================== ACWB host
int cwb_train_acwb_general(cwb_ctx* c, const double* Y, int32_t B, double nu, double gamma, int32_t M,
                           double* offset_out, double* theta_f_out, double* theta_h_out, int32_t* k_trace,
                           int32_t* kcor_trace, double* sse_trace, double* risk_trace, cudaStream_t s) {
    int rc = ensure_ws(c, 2 * B, s);
    if (rc) return rc;
    cwb_train_ws& w = c->ws;
    const int Bp = w.Bp, Bq = (B + 31) / 32 * 32;
    const int nblk = (int)((c->n + kRowsH6 - 1) / kRowsH6);
    const size_t need = sizeof(double) * (2 * (size_t)c->n * Bq + 3 * (size_t)nblk * Bq + Bq);
    if (w.acwb_bytes < need) {
        cwb_release(w.acwb, s);
        w.acwb = nullptr;
        w.acwb_bytes = 0;
        if (cwb_alloc((void**)&w.acwb, need, s) != cudaSuccess)
            return cwb_set_error(c, CWB_ENOMEM, "ACWB workspace allocation failed");
        w.acwb_bytes = need;
    }
    double* F = w.acwb;
    double* H = F + (size_t)c->n * Bq;
    double* part = H + (size_t)c->n * Bq;
    double* off_ws = part + 3 * (size_t)nblk * Bq;
    // line 2: f0 = mean(y); f = h = g = f0; r^[1] = c^[1] = y - f0
    rc = column_stats(c, Y, B, true, off_ws, w.rr, offset_out, s);
    if (rc) return rc;
    dim3 gt((unsigned)((c->n + 31) / 32), Bp / 32);
    k_tr_in<<<gt, dim3(32, 8), 0, s>>>(Y, c->n, B, Bp, off_ws, nullptr, w.Rt);
    k_acwb_init<<<dim3((unsigned)std::min<int64_t>(2048, (c->n + 7) / 8), Bq / 32), 256, 0, s>>>(w.Rt, F, H, c->n, B,
                                                                                                  Bp, Bq);
    cudaMemcpyAsync(w.rr + B, w.rr, sizeof(double) * B, cudaMemcpyDeviceToDevice, s);
    const size_t nagg = (size_t)B * c->K * c->d;
    k_zero<<<(unsigned)std::min((size_t)1184, (nagg + 255) / 256 + 1), 256, 0, s>>>(theta_f_out, nagg);
    k_zero<<<(unsigned)std::min((size_t)1184, (nagg + 255) / 256 + 1), 256, 0, s>>>(theta_h_out, nagg);
    c->launches += 5;
    for (int m = 1; m <= M; m++) {
        const double vt = 2.0 / (double)(m + 1);              // line 4
        const double eta = gamma * nu / vt;                   // line 15
        const double vt1 = 2.0 / (double)(m + 2);             // next iteration's combination
        const double a1 = (double)(m + 1) / (double)(m + 2);  // next iteration's correction weight
        h1(c, w.Rt, Bp, c->K, c->n_star, c->off, c->perm, c->perm_bytes, w.U, s);  // lines 7 and 14: binMatVec
        k_h234<<<dim3(c->K, Bp / 32), 256, 0, s>>>(w.U, Bp, c->n_star, c->d, c->ZT, c->W, c->lwin, c->Ainv, c->G,
                                                    w.theta, w.delta);
        k_acwb_select<<<(B + 127) / 128, 128, 0, s>>>(w.delta, w.theta, w.rr, c->K, c->d, B, Bp, nu, vt, eta, m - 1,
                                                      w.kstar, theta_f_out, theta_h_out, k_trace, kcor_trace,
                                                      sse_trace);
        k_zhat<<<dim3((c->n_star + 7) / 8, Bp / 32), 256, 0, s>>>(w.kstar, w.theta, c->zj0, c->Zs, c->n_star, c->d,
                                                                  2 * B, Bp, nu, B, 1.0, w.zhat);
        dim3 g6(nblk, Bq / 32);
        if (c->idx_bytes == 1)
            k_acwb_update<uint8_t><<<g6, 256, 0, s>>>(w.Rt, F, H, c->n, B, Bp, Bq, w.kstar, (const uint8_t*)c->idx,
                                                      w.zhat, eta, vt1, a1, part);
        else
            k_acwb_update<uint16_t><<<g6, 256, 0, s>>>(w.Rt, F, H, c->n, B, Bp, Bq, w.kstar, (const uint16_t*)c->idx,
                                                       w.zhat, eta, vt1, a1, part);
        k_acwb_rr<<<(B + 127) / 128, 128, 0, s>>>(part, nblk, B, Bq, c->n, m - 1, w.rr, risk_trace);
        c->launches += 6;
    }
    return cwb_check_launch(c, "ACWB kernels");
}

// ===================================================================== HCWB host
int cwb_train_hcwb_general(cwb_ctx* c, const double* Y, int32_t B, const uint8_t* val_mask, double nu, double gamma,
                           int32_t pat0, int32_t M, double* offset_out, double* theta_f_out, int32_t* k_trace,
                           int32_t* kcor_trace, double* sse_trace, double* risk_trace, double* val_risk_trace,
                           int32_t* switch_iter, cudaStream_t s) {
    int rc = ensure_ws(c, 2 * B, s);
    if (rc) return rc;
    cwb_train_ws& w = c->ws;
    const int Bp = w.Bp, Bq = (B + 31) / 32 * 32;
    const int K = c->K, ns = c->n_star, d = c->d;
    const int nblk = (int)((c->n + kRowsH6 - 1) / kRowsH6);
    // F, H (n x Bq), partials (4 x nblk x Bq), offsets, theta_h (B x K x d), vprev, counts,
    // G_tr, Ainv_tr (K x d x d), cnt_tr (K x n*), phase, pat (ints)
    const size_t dbl = 2 * (size_t)c->n * Bq + 4 * (size_t)nblk * Bq + Bq + (size_t)B * K * d + Bq + 2 +
                       2 * (size_t)K * d * d + 4 * (size_t)K * d;
    const size_t need = sizeof(double) * dbl + sizeof(uint32_t) * (size_t)K * ns + 2 * sizeof(int32_t) * Bq;
    if (w.acwb_bytes < need) {
        cwb_release(w.acwb, s);
        w.acwb = nullptr;
        w.acwb_bytes = 0;
        if (cwb_alloc((void**)&w.acwb, need, s) != cudaSuccess)
            return cwb_set_error(c, CWB_ENOMEM, "HCWB workspace allocation failed");
        w.acwb_bytes = need;
    }
    double* F = w.acwb;
    double* H = F + (size_t)c->n * Bq;
    double* part = H + (size_t)c->n * Bq;
    double* off_ws = part + 4 * (size_t)nblk * Bq;
    double* th = off_ws + Bq;
    double* vprev = th + (size_t)B * K * d;
    double* cnt = vprev + Bq;
    double* G_tr = cnt + 2;
    double* Ainv_tr = G_tr + (size_t)K * d * d;
    double* Cb_tr = Ainv_tr + (size_t)K * d * d;
    uint32_t* cnt_tr = (uint32_t*)(Cb_tr + (size_t)K * d * 4);
    int32_t* phase = (int32_t*)(cnt_tr + (size_t)K * ns);
    int32_t* pat = phase + Bq;
    k_mask_count<<<1, 1024, 0, s>>>(val_mask, c->n, cnt, c->d_status);
    rc = cwb_launch_masked_pool(c, val_mask, cnt_tr, G_tr, Ainv_tr, s, Cb_tr);
    if (rc) return rc;
    if (c->path != 2) {  // the whole run in one persistent kernel when it fits (cwb_fused.cu, HC mode)
        bool launched = false;
        rc = cwb_train_hcwb_fused(c, Y, B, val_mask, Ainv_tr, Cb_tr, nu, gamma, pat0, M, offset_out, theta_f_out,
                                  k_trace, kcor_trace, sse_trace, risk_trace, val_risk_trace, switch_iter, s,
                                  &launched);
        if (rc || launched) return rc;
        if (c->path == 1) {  // a device-side error (e.g. the mask check above) stopped the plan: report it first
            const int st = cwb_status(c);
            if (st) return st;
            return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_train_hcwb: fused path does not fit");
        }
    }
    cudaMemsetAsync(phase, 0, sizeof(int32_t) * 2 * Bq, s);
    // f0 = mean of the training targets (Alg. 2 line 2 on D_train); rr = sum over training rows
    rc = column_stats(c, Y, B, true, off_ws, w.rr, offset_out, s, val_mask, 0, cnt);
    if (rc) return rc;
    {   // validation risk of f0: sum over validation rows of (y - f0)^2 / (2 n_val)
        const int nb = (int)((c->n + kColRows - 1) / kColRows);
        k_colsum<<<dim3(nb, B), 256, 0, s>>>(Y, c->n, off_ws, true, w.colpart, c->d_status, val_mask, 1);
        k_center_fin<<<(B + 127) / 128, 128, 0, s>>>(w.colpart, nb, B, c->n, 1, vprev, nullptr);
        c->launches += 2;
    }
    cudaMemcpyAsync(w.rr + B, w.rr, sizeof(double) * B, cudaMemcpyDeviceToDevice, s);
    dim3 gt((unsigned)((c->n + 31) / 32), Bp / 32);
    k_tr_in<<<gt, dim3(32, 8), 0, s>>>(Y, c->n, B, Bp, off_ws, nullptr, w.Rt);
    k_hcwb_init<<<dim3((unsigned)std::min<int64_t>(2048, (c->n + 7) / 8), Bq / 32), 256, 0, s>>>(w.Rt, F, H, val_mask,
                                                                                                  c->n, B, Bp, Bq);
    const size_t nagg = (size_t)B * K * d;
    k_zero<<<(unsigned)std::min((size_t)1184, (nagg + 255) / 256 + 1), 256, 0, s>>>(theta_f_out, nagg);
    k_zero<<<(unsigned)std::min((size_t)1184, (nagg + 255) / 256 + 1), 256, 0, s>>>(th, nagg);
    c->launches += 5;
    // vprev holds sum (y - f0)^2 over validation rows: scale by 1 / (2 n_val) once
    k_hcwb_scale_vprev<<<(B + 127) / 128, 128, 0, s>>>(vprev, cnt, B);
    if (switch_iter) k_fill_int<<<(B + 127) / 128, 128, 0, s>>>(switch_iter, B, M);
    c->launches += 2;
    for (int m = 0; m < M; m++) {
        // ACWB iteration index ma = m + 1 while a replication is in phase 0
        const double vt = 2.0 / (double)(m + 2);
        const double eta = gamma * nu / vt;
        const double vt1 = 2.0 / (double)(m + 3);
        const double a1 = (double)(m + 2) / (double)(m + 3);
        h1(c, w.Rt, Bp, K, ns, c->off, c->perm, c->perm_bytes, w.U, s);
        k_h234<<<dim3(K, Bp / 32), 256, 0, s>>>(w.U, Bp, ns, d, c->ZT, c->W, c->lwin, Ainv_tr, G_tr, w.theta, w.delta,
                                                c->Ainv, c->G, phase, B);
        k_hcwb_select<<<(B + 127) / 128, 128, 0, s>>>(w.delta, w.theta, w.rr, phase, K, d, B, Bp, nu, vt, eta, m,
                                                      w.kstar, theta_f_out, th, k_trace, kcor_trace, sse_trace);
        k_zhat<<<dim3((ns + 7) / 8, Bp / 32), 256, 0, s>>>(w.kstar, w.theta, c->zj0, c->Zs, ns, d, 2 * B, Bp, nu, B,
                                                           1.0, w.zhat);
        dim3 g6(nblk, Bq / 32);
        if (c->idx_bytes == 1)
            k_hcwb_update<uint8_t><<<g6, 256, 0, s>>>(F, H, val_mask, c->n, B, Bp, Bq, phase, w.kstar,
                                                      (const uint8_t*)c->idx, w.zhat, vt, eta, part);
        else
            k_hcwb_update<uint16_t><<<g6, 256, 0, s>>>(F, H, val_mask, c->n, B, Bp, Bq, phase, w.kstar,
                                                       (const uint16_t*)c->idx, w.zhat, vt, eta, part);
        k_hcwb_decide<<<(B + 127) / 128, 128, 0, s>>>(part, nblk, B, Bq, c->n, cnt, m, pat0, phase, pat, vprev,
                                                      switch_iter, risk_trace, val_risk_trace);
        if (c->idx_bytes == 1)
            k_hcwb_prepare<uint8_t><<<g6, 256, 0, s>>>(w.Rt, F, H, val_mask, c->n, B, Bp, Bq, phase, w.kstar,
                                                       (const uint8_t*)c->idx, w.zhat, vt1, a1, part);
        else
            k_hcwb_prepare<uint16_t><<<g6, 256, 0, s>>>(w.Rt, F, H, val_mask, c->n, B, Bp, Bq, phase, w.kstar,
                                                        (const uint16_t*)c->idx, w.zhat, vt1, a1, part);
        k_hcwb_rr<<<(B + 127) / 128, 128, 0, s>>>(part, nblk, B, Bq, w.rr);
        c->launches += 8;
    }
    return cwb_check_launch(c, "HCWB kernels");
}

// ===================================================================== cross-Gram path (cwb_set_path 3)
// SURVEY Sec. 7.3 item 3, an exact reformulation of Alg. 1 supp. for the L2 loss with fixed weights.  With
// Z_k the n x d design of learner k (row i = Zb_k[idx_k(i)]), s_k = Z_k^T r and the
// cached fit theta_k = A_k^-1 s_k (A_k = G_k + lambda_k D):
//   r^[m] = r^[m-1] - nu Z_k* theta*
//   => theta_k^[m] = theta_k^[m-1] - nu W_k,k* theta*,   W_k,k' = A_k^-1 (Z_k^T Z_k')
//      r^T r ^[m] = r^T r - 2 nu theta*^T s_k* + nu^2 theta*^T G_k* theta* = r^T r - nu delta* - nu (1 - nu) theta*^T G_k* theta*
// (delta = 2 theta^T s - theta^T G theta), so after one binMatVec pass for theta^[0] (H1-H3 on the
// initial residuals) an iteration costs O(K d^2) per replication instead of O(n).  delta_k = |C_k^T theta_k|^2,
// SSE_k = r^T r - delta_k and the argmin are those of the direct path (H4, H5).  The cross Gram Z^T Z
// (K d x K d) is itself binMatVec-shaped: with P = [Z_1 ... Z_K] (n x K d, gathered basis rows),
// (Z_k^T Z)[a][.] = sum_l Zb_k[l][a] U_k[l][.], U_k[l][.] = sum_{i: idx_k(i) = l} P[i][.] -- H1 and the H2
// projection on the K d "columns" of P.
namespace {

// P[i - r0][k d + a] = Zb_k[idx_k(i)][a] for the rows i in [r0, r1) (4 non-zeros per learner block; columns
// >= K d are 0)
template <typename IdxT>
__global__ void k_gram_P(const IdxT* __restrict__ idx, int64_t n, int64_t r0, int64_t r1, int K, int ns, int d, int ld,
                         const int32_t* __restrict__ zj0, const double* __restrict__ Zs, double* __restrict__ P) {
    const int64_t tot = (r1 - r0) * ld;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t il = e / ld, i = r0 + il;
        const int col = (int)(e - il * ld);
        double v = 0.0;
        if (col < K * d) {
            const int k = col / d, a = col - k * d;
            const int l = (int)idx[(size_t)k * n + i];
            const int t = a - zj0[(size_t)k * ns + l];
            if (t >= 0 && t < CWB_SPW) v = Zs[((size_t)k * ns + l) * CWB_SPW + t];
        }
        P[e] = v;
    }
}

// Wt[(k' d + b) ld + k d + a] = (A_k^-1 Z_k^T Z_k')[a][b] = sum_c A_k^-1[a][c] xg[(k' d + b) ld + k d + c]
// (xg symmetric): row (k', b) of Wt is what an iteration with k* = k' reads, contiguous in (k, a)
__global__ void k_gram_w(const double* __restrict__ xg, const double* __restrict__ Ainv, int K, int d, int ld,
                         double* __restrict__ Wt) {
    const int row = blockIdx.x;  // k' d + b
    const double* xr = xg + (size_t)row * ld;
    for (int q = threadIdx.x; q < ld; q += blockDim.x) {
        double v = 0.0;
        if (q < K * d) {
            const int k = q / d, a = q - k * d;
            const double* Ai = Ainv + ((size_t)k * d + a) * d;
            for (int c = 0; c < d; c++) v += Ai[c] * xr[k * d + c];
        }
        Wt[(size_t)row * ld + q] = v;
    }
}

// One CTA per replication b, all M iterations.  Shared: theta of every learner (K d), delta (K), theta* (d);
// C (the band factor of G + 2 lambda D, K d 4) is read through L1.  th0: [K d][Bp] (k_h234 layout), rr0: [Bp].  Per iteration:
//   A  warp per learner: c = C_k^T theta_k (the band, 3 shuffles), delta_k = |c|^2                   (H4)
//   B  warp 0: k* = argmax delta (lowest k on ties), SSE, theta_agg[k*] += nu theta* (P:L838),
//      t2 = theta*^T G_k* theta*, r^T r -= nu delta* + nu (1 - nu) t2, traces
//   C  every thread: theta[q] -= nu sum_b Wt[(k* d + b) ld + q] theta*[b]
__global__ void __launch_bounds__(256) k_gram_train(
    const double* __restrict__ th0, int Bp, const double* __restrict__ rr0, const double* __restrict__ Wt, int ld,
    const double* __restrict__ Cb, const double* __restrict__ G, int K, int d, int64_t n, double nu, int M, int B,
    double* __restrict__ agg, int32_t* __restrict__ k_trace, double* __restrict__ sse_trace,
    double* __restrict__ risk_trace) {
    extern __shared__ double gsm[];
    const int Kd = K * d;
    double* th = gsm;              // K d
    double* de = th + Kd;          // K   (the band factor stays in global memory: L1-resident, shared by all CTAs)
    __shared__ double s_rr, s_ts[CWB_MAX_D];
    __shared__ int s_k;
    const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
    for (int q = tid; q < Kd; q += blockDim.x) th[q] = th0[(size_t)q * Bp + b];
    if (tid == 0) s_rr = rr0[b];
    double* ag = agg + (size_t)b * Kd;
    for (int q = tid; q < Kd; q += blockDim.x) ag[q] = 0.0;
    __syncthreads();
    for (int m = 0; m < M; m++) {
        CWB_JIT(m * 4 + 0);
        // A: delta_k = |C_k^T theta_k|^2, c_j = sum_{i<4} C[j+i][j] theta[j+i]
        for (int k = w; k < K; k += nw) {
            const double t = lane < d ? th[k * d + lane] : 0.0;
            double c = 0.0;
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const double tj = __shfl_down_sync(0xffffffffu, t, i);
                if (lane + i < d && lane < d) c += __ldg(Cb + (k * d + lane) * 4 + i) * tj;
            }
            const double dl = warp_sum(lane < d ? c * c : 0.0);
            if (lane == 0) de[k] = dl;
        }
        __syncthreads();
        CWB_JIT(m * 4 + 1);
        // B: H5 and the scalar updates
        if (w == 0) {
            int kb = -1;
            double best = -1.0;
            for (int k = lane; k < K; k += 32) {  // ascending k per lane: strict > keeps the lowest
                const double v = de[k];
                if (kb < 0 || v > best) { best = v; kb = k; }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int ok = __shfl_xor_sync(0xffffffffu, kb, o);
                if (ok >= 0 && (kb < 0 || ob > best || (ob == best && ok < kb))) { best = ob; kb = ok; }
            }
            const int ks = kb;
            const double tj = lane < d ? th[ks * d + lane] : 0.0;
            double g = 0.0;
            if (lane < d) {
                const double* Gk = G + ((size_t)ks * d + lane) * d;
                for (int jp = max(0, lane - (CWB_SPW - 1)); jp <= min(d - 1, lane + CWB_SPW - 1); jp++)
                    g += Gk[jp] * th[ks * d + jp];   // G banded (|j - j'| <= 3)
                s_ts[lane] = tj;
                ag[ks * d + lane] += nu * tj;
            }
            const double t2 = warp_sum(tj * g);
            if (lane == 0) {
                const double rr = s_rr;
                const double rrn = rr - nu * best - nu * (1.0 - nu) * t2;
                if (k_trace) k_trace[(size_t)m * B + b] = ks;
                if (sse_trace) sse_trace[(size_t)m * B + b] = rr - best;
                if (risk_trace) risk_trace[(size_t)m * B + b] = rrn / (2.0 * (double)n);
                s_rr = rrn;
                s_k = ks;
            }
        }
        __syncthreads();
        CWB_JIT(m * 4 + 2);
        // C: theta_k -= nu W_k,k* theta*
        {
            const int ks = s_k;
            const double* wr = Wt + (size_t)ks * d * ld;
            for (int q = tid; q < Kd; q += blockDim.x) {
                double u0 = 0.0, u1 = 0.0;
                int bb = 0;
                for (; bb + 8 <= d; bb += 8) {  // eight row loads of W^T in flight
                    double w8[8];
#pragma unroll
                    for (int x = 0; x < 8; x++) w8[x] = __ldg(wr + (size_t)(bb + x) * ld + q);
#pragma unroll
                    for (int x = 0; x < 8; x += 2) {
                        u0 = fma(w8[x], s_ts[bb + x], u0);
                        u1 = fma(w8[x + 1], s_ts[bb + x + 1], u1);
                    }
                }
                for (; bb < d; bb++) u0 = fma(__ldg(wr + (size_t)bb * ld + q), s_ts[bb], u0);
                th[q] -= nu * (u0 + u1);
            }
        }
        __syncthreads();
    }
}

}  // namespace

// idxT[i][k] = idx_k(i) as uint16, row-major with Kp (a multiple of 32) learners per row: the bins of one row
// of all learners are contiguous (one or a few sectors), tile transpose through shared memory
template <typename IdxT>
__global__ void k_idx_rowmajor(const IdxT* __restrict__ idx, int64_t n, int K, int Kp, uint16_t* __restrict__ idxT) {
    __shared__ uint16_t tile[32][33];
    const int64_t i0 = (int64_t)blockIdx.x * 32;
    const int k0 = blockIdx.y * 32;
    for (int m = threadIdx.y; m < 32; m += blockDim.y) {
        const int k = k0 + m;
        const int64_t i = i0 + threadIdx.x;
        tile[m][threadIdx.x] = (k < K && i < n) ? (uint16_t)idx[(size_t)k * n + i] : (uint16_t)0;
    }
    __syncthreads();
    for (int m = threadIdx.y; m < 32; m += blockDim.y) {
        const int64_t i = i0 + m;
        if (i < n) idxT[(size_t)i * Kp + k0 + threadIdx.x] = tile[threadIdx.x][m];
    }
}

// idxP[slot(k, k')][j] = idx_k'(perm_k[j]) for the learners k of the launch (blockIdx.y -> k = kb0 + y) and every
// k' >= k; slot(k, k') = sum_{k'' in [kb0, k)} (K - k'') + k' - k.  A warp takes 32 consecutive positions j: it
// reads the 32 rows' learner chunks from idxT (lanes over k', contiguous) into a shared tile and writes them
// back with lanes over j (contiguous in idxP).
template <typename PermT>
__global__ void __launch_bounds__(256) k_gram_pregather(const uint16_t* __restrict__ idxT, const PermT* __restrict__ perm,
                                                         int64_t n, int K, int Kp, int kb0,
                                                         uint16_t* __restrict__ idxP) {
    __shared__ uint16_t tile[8][32][34];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int k = kb0 + blockIdx.y;
    size_t slot0 = 0;
    for (int kk = kb0; kk < k; kk++) slot0 += (size_t)(K - kk);
    const PermT* pk = perm + (size_t)k * n;
    const int64_t ntile = (n + 31) / 32;
    for (int64_t t = (int64_t)blockIdx.x * 8 + w; t < ntile; t += (int64_t)gridDim.x * 8) {
        const int64_t j0 = t * 32;
        const int64_t jm = j0 + lane;
        const uint32_t irow = jm < n ? (uint32_t)pk[jm] : 0u;  // row ids fit 32 bits (off is int32)
        // learner chunks start at k (not at a multiple of 32): no lanes spent on learners k' < k
        for (int c0 = k; c0 < K; c0 += 32) {
            const int cl = min(c0 + lane, Kp - 1);  // (columns >= K are padding; never written out)
            uint16_t vals[32];  // all 32 row loads in flight before the tile stores
#pragma unroll
            for (int r = 0; r < 32; r++) {
                const uint32_t ir = __shfl_sync(0xffffffffu, irow, r);
                vals[r] = idxT[(size_t)ir * Kp + cl];
            }
#pragma unroll
            for (int r = 0; r < 32; r++) tile[w][lane][r] = vals[r];
            __syncwarp();
            const int qn = min(32, K - c0);
            for (int q = 0; q < qn; q++)
                if (jm < n) idxP[(slot0 + (size_t)(c0 + q - k)) * n + jm] = tile[w][q][lane];
            __syncwarp();
        }
    }
}

// Cross-Gram block of a pair of learners through their joint bin counts -- binMatMat's "counts times
// design-point products" (G_k = Zb_k^T diag(c) Zb_k with c the bin counts) for two index vectors:
//   (Z_k^T Z_k')[a][b] = sum_{l, l'} C[l][l'] Zb_k[l][a] Zb_k'[l'][b],   C[l][l'] = #{i : idx_k(i) = l, idx_k'(i) = l'}
// (rows of one (l, l') cell have identical basis rows in both learners).  One CTA per pair k <= k',
// bins of k in tiles of TL: the tile's rows are contiguous in the bin inversion perm_k; their idx_k' values are
// counted into C[tile][n*] (u32 shared-memory atomics: integer, order-free), then
//   V[l][b] = sum_{l' in window of b} C[l][l'] Zb_k'[l'][b]      (window-major basis ZT, lwin)
//   acc[a][b] += sum_{l in tile, in window of a} Zb_k[l][a] V[l][b]   (thread (a, b), tiles ascending: fixed order)
// The idx_k' values of the tile's rows are read from idxP: for every pair slot of the launch, idx_k' permuted into
// the bin order of k (idxP[slot][j] = idx_k'(perm_k[j]), k_gram_pregather), so the counting pass is a coalesced
// stream (a per-row gather of 2-byte values from idx_k' costs a 32-byte sector each and, at R4, thrashes L2).
__global__ void __launch_bounds__(1024, 1) k_gram_joint(const uint16_t* __restrict__ idxP, int kb0,
                                                         const int32_t* __restrict__ off, int64_t n, int K, int ns,
                                                         int d, int TL, const double* __restrict__ ZT, int W,
                                                         const int32_t* __restrict__ lwin,
                                                         const double* __restrict__ Zb, const double* __restrict__ G,
                                                         double* __restrict__ xg, int ld) {
    extern __shared__ __align__(16) unsigned char gsm[];
    const int hs = ns | 1;  // odd row stride: the lanes of stage 1 (consecutive bins of k) hit distinct banks
    uint32_t* hist = reinterpret_cast<uint32_t*>(gsm);                                          // [TL][hs]
    double* V = reinterpret_cast<double*>(gsm + (((size_t)TL * hs * 4 + 15) & ~(size_t)15));    // [TL][d]
    double* zks = V + (size_t)TL * d;             // [TL][d]  Zb_k rows of the tile
    double* zps = zks + (size_t)TL * d;           // [W][d]   window-major basis of k' (read every tile)
    int32_t* oks = reinterpret_cast<int32_t*>(zps + (size_t)W * d);                              // [TL + 1] bin starts
    int k = kb0, kp = 0;
    {   // slot of the launch -> (k, k'), k' >= k (row k of the upper triangle holds K - k pairs), k from kb0
        int rem = blockIdx.x;
        while (rem >= K - k) { rem -= K - k; k++; }
        kp = k + rem;
    }
    const uint16_t* ip = idxP + (size_t)blockIdx.x * n;
    const int32_t* ok = off + (size_t)k * (ns + 1);
    const double* ztp = ZT + (size_t)kp * W * d;
    const double* zbk = Zb + (size_t)k * ns * d;
    const int32_t* lwp = lwin + (size_t)kp * d * 2;
    const int tid = threadIdx.x;
    const bool own = tid < d * d;  // d <= CWB_MAX_D = 32: d^2 <= blockDim
    const int a = tid / d, b = tid - a * d;
    if (kp == k) {  // Z_k^T Z_k = G_k (binMatMat, I6): already in the pool
        if (own) xg[((size_t)k * d + a) * ld + (size_t)kp * d + b] = G[(size_t)k * d * d + tid];
        return;
    }
    for (int e = tid; e < W * d; e += blockDim.x) zps[e] = ztp[e];
    double acc = 0.0;
    for (int t0 = 0; t0 < ns; t0 += TL) {
        const int t1 = min(ns, t0 + TL);
        const int tlc = t1 - t0;
        for (int e = tid; e < tlc * hs; e += blockDim.x) hist[e] = 0u;
        for (int e = tid; e <= tlc; e += blockDim.x) oks[e] = ok[t0 + e];
        for (int e = tid; e < tlc * d; e += blockDim.x) zks[e] = zbk[(size_t)t0 * d + e];
        __syncthreads();
        // the tile's rows are contiguous in the bin order of k: threads stride over aligned groups of 8 rows (one
        // 16-byte load each, four in flight: a tile costs one or two DRAM round trips), balanced whatever the bin
        // sizes; each thread's bin pointer only moves forward.  Groups may start up to 7 rows before the tile /
        // end after it (masked; idxP is allocated with 16 bytes of slack on both sides).
        {
            const int jb = oks[0], je = oks[tlc];
            const int sh = (int)(((16 - ((uintptr_t)ip & 15)) & 15) >> 1);  // rows to the first 16-byte boundary
            const int g0 = (jb - sh + 8) / 8 - 1, g1 = (je - sh + 7) / 8;   // groups [g0, g1) cover [jb, je)
            int l = 0;
            for (int g = g0 + tid; g < g1; g += 4 * 1024) {
                uint4 v[4];
#pragma unroll
                for (int u = 0; u < 4; u++)
                    if (g + u * 1024 < g1) v[u] = *reinterpret_cast<const uint4*>(ip + sh + 8 * (int64_t)(g + u * 1024));
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    if (g + u * 1024 >= g1) break;
                    const int r0 = sh + 8 * (g + u * 1024);
                    const uint32_t wv[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
                    while (r0 >= oks[l + 1]) l++;  // (r0 < jb on the first group: l stays 0)
                    if (r0 >= jb && r0 + 7 < min(je, oks[l + 1])) {  // the whole group inside one bin of the tile
                        uint32_t* hl = hist + (size_t)l * hs;
#pragma unroll
                        for (int e = 0; e < 8; e++)
                            atomicAdd(&hl[(e & 1) ? (wv[e >> 1] >> 16) : (wv[e >> 1] & 0xffffu)], 1u);
                    } else {
#pragma unroll
                        for (int e = 0; e < 8; e++) {
                            const int jj = r0 + e;
                            if (jj < jb || jj >= je) continue;
                            const uint32_t cv = (e & 1) ? (wv[e >> 1] >> 16) : (wv[e >> 1] & 0xffffu);
                            while (jj >= oks[l + 1]) l++;
                            atomicAdd(&hist[(size_t)l * hs + cv], 1u);
                        }
                    }
                }
            }
        }
        __syncthreads();
        for (int e = tid; e < tlc * d; e += blockDim.x) {  // lanes: consecutive bins of k, one basis b of k'
            const int bb = e / tlc, tl = e - bb * tlc;
            const int lb = lwp[bb * 2], len = lwp[bb * 2 + 1] - lb;
            const uint32_t* hl = hist + (size_t)tl * hs + lb;
            const double* zt = zps + bb;
            double sacc = 0.0;
            // u32 -> double by the 2^52 bit pattern and one subtraction (exact; the FP64 pipe instead of I2F.F64)
            for (int x = 0; x < len; x++)
                sacc = fma(__hiloint2double(0x43300000, (int)hl[x]) - 4503599627370496.0, zt[x * d], sacc);
            V[tl * d + bb] = sacc;
        }
        __syncthreads();
        if (own)  // Zb_k[l][a] is 0 outside the window of a: the whole tile in bin order
            for (int tl = 0; tl < tlc; tl++) acc = fma(zks[tl * d + a], V[tl * d + b], acc);
        __syncthreads();
    }
    if (own) xg[((size_t)k * d + a) * ld + (size_t)kp * d + b] = acc;
}

// lower blocks of the symmetric cross Gram from the upper ones: xg[(k,a)][(k',b)] = xg[(k',b)][(k,a)], k' < k
__global__ void k_gram_sym(double* __restrict__ xg, int K, int d, int ld) {
    const int row = blockIdx.x, k = row / d;  // row = k d + a
    for (int q = threadIdx.x; q < k * d; q += blockDim.x) xg[(size_t)row * ld + q] = xg[(size_t)q * ld + row];
}

// builds the cross Gram of the pool's K learners and Wt = (A^-1 Z^T Z)^T rows once per pool (c->xg)
static int gram_build(cwb_ctx* c, cudaStream_t s) {
    if (c->xg) return CWB_OK;
    const int K = c->K, d = c->d, ns = c->n_star;
    const int ld = (K * d + 63) / 64 * 64;  // whole 64-column tiles: the wide H1
    const int64_t n = c->n;
    double *P = nullptr, *U = nullptr, *xg = nullptr, *Wt = nullptr;
    // joint-bin-count build (k_gram_joint) when a tile of the count table fits shared memory; CWB_GRAM_JOINT=0
    // keeps the gathered-basis build below (the A/B and the fallback for very large n*)
    static const int joint_on = getenv("CWB_GRAM_JOINT") ? atoi(getenv("CWB_GRAM_JOINT")) : 1;
    {
        int dev = 0, optin = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        const size_t per_bin = (size_t)(ns | 1) * 4 + (size_t)d * 16 + 4;
        const size_t budget = (size_t)std::max<int64_t>(0, (int64_t)optin - 2048 - (int64_t)c->W * d * 8);
        int TL = (int)std::min<size_t>((size_t)ns, budget > 64 ? (budget - 64) / per_bin : 0);
        if (joint_on && TL >= 1 && d * d <= 1024) {
            // whole rounds of the 1024 threads in the (bin, basis) contraction; then equal tiles
            const int q = std::max(1, 1024 / d);
            if (TL >= q && TL < ns) TL = TL / q * q;
            else if (TL < ns) TL = (ns + (ns + TL - 1) / TL - 1) / ((ns + TL - 1) / TL);
            const size_t smem = (((size_t)TL * (ns | 1) * 4 + 15) & ~(size_t)15) + (size_t)TL * d * 16 +
                                (size_t)c->W * d * 8 + (size_t)(TL + 1) * 4 + 16;
            bool ok2 = cwb_alloc((void**)&xg, sizeof(double) * (size_t)K * d * ld, s) == cudaSuccess;
            ok2 &= cwb_alloc((void**)&Wt, sizeof(double) * (size_t)K * d * ld, s) == cudaSuccess;
            if (!ok2) {
                cwb_release(xg, s); cwb_release(Wt, s);
                return cwb_set_error(c, CWB_ENOMEM, "cross-Gram workspace allocation failed");
            }
            CWB_CUDA_TRY(c, cudaMemsetAsync(xg, 0, sizeof(double) * (size_t)K * d * ld, s));
            // idx row-major (all learners' bins of a row adjacent), then per batch of learners k: the permuted
            // index rows of its pairs (at most ~1 GiB at a time) and one CTA per pair
            const int Kp = (K + 31) / 32 * 32;
            const size_t slot_cap = std::max<size_t>((size_t)K, ((size_t)1 << 30) / ((size_t)n * 2));
            uint16_t *idxT = nullptr, *idxP = nullptr;
            const size_t slots_all = (size_t)K * (K + 1) / 2;
            ok2 = cwb_alloc((void**)&idxT, sizeof(uint16_t) * (size_t)n * Kp, s) == cudaSuccess;
            uint16_t* idxP_base = nullptr;  // 16 bytes of slack before and after the slots (k_gram_joint's aligned loads)
            ok2 &= cwb_alloc((void**)&idxP_base, sizeof(uint16_t) * ((size_t)n * std::min(slot_cap, slots_all) + 16), s) == cudaSuccess;
            idxP = idxP_base ? idxP_base + 8 : nullptr;
            if (!ok2) {
                cwb_release(idxT, s); cwb_release(idxP_base, s); cwb_release(xg, s); cwb_release(Wt, s);
                return cwb_set_error(c, CWB_ENOMEM, "cross-Gram workspace allocation failed");
            }
            {
                dim3 g((unsigned)((n + 31) / 32), (unsigned)(Kp / 32));
                if (c->idx_bytes == 1) k_idx_rowmajor<uint8_t><<<g, dim3(32, 8), 0, s>>>((const uint8_t*)c->idx, n, K, Kp, idxT);
                else k_idx_rowmajor<uint16_t><<<g, dim3(32, 8), 0, s>>>((const uint16_t*)c->idx, n, K, Kp, idxT);
                c->launches++;
            }
            CWB_CUDA_TRY(c, cudaFuncSetAttribute(k_gram_joint, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            for (int kb0 = 0; kb0 < K;) {
                int kb1 = kb0;
                size_t slots = 0;
                while (kb1 < K && (kb1 == kb0 || slots + (size_t)(K - kb1) <= slot_cap)) slots += (size_t)(K - kb1++);
                const unsigned gx = (unsigned)std::min<int64_t>(((n + 31) / 32 + 7) / 8, (int64_t)cwb_num_sms() * 8);
                dim3 gp(gx, (unsigned)(kb1 - kb0));
                if (c->perm_bytes == 2)
                    k_gram_pregather<uint16_t><<<gp, 256, 0, s>>>(idxT, (const uint16_t*)c->perm, n, K, Kp, kb0, idxP);
                else
                    k_gram_pregather<uint32_t><<<gp, 256, 0, s>>>(idxT, (const uint32_t*)c->perm, n, K, Kp, kb0, idxP);
                k_gram_joint<<<(unsigned)slots, 1024, smem, s>>>(idxP, kb0, c->off, n, K, ns, d, TL, c->ZT, c->W,
                                                                 c->lwin, c->Zb, c->G, xg, ld);
                c->launches += 2;
                kb0 = kb1;
            }
            CWB_CUDA_TRY(c, cudaGetLastError());
            cwb_release(idxT, s);
            cwb_release(idxP_base, s);
            k_gram_sym<<<K * d, 256, 0, s>>>(xg, K, d, ld);
            k_gram_w<<<K * d, 256, 0, s>>>(xg, c->Ainv, K, d, ld, Wt);
            c->launches += 3;
            cwb_release(xg, s);
            c->xg = Wt;
            c->xg_ld = ld;
            return cwb_check_launch(c, "cross-Gram kernels (joint bin counts)");
        }
    }
    // the gathered basis P is built one H1 row chunk at a time (n x ld would be 16 GB at R4)
    int nch = 1;
    const int64_t CR = h1_chunk_plan(c, c->h1_wide ? 512 : 256, c->off, K, ns, &nch, s);
    if (CR < 0) return c->status ? c->status : CWB_ENOMEM;
    const int64_t prow = CR > 0 ? CR : n;
    bool ok = cwb_alloc((void**)&P, sizeof(double) * (size_t)prow * ld, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&U, sizeof(double) * (size_t)K * ns * ld, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&xg, sizeof(double) * (size_t)K * d * ld, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&Wt, sizeof(double) * (size_t)K * d * ld, s) == cudaSuccess;
    if (!ok) {
        cwb_release(P, s); cwb_release(U, s); cwb_release(xg, s); cwb_release(Wt, s);
        return cwb_set_error(c, CWB_ENOMEM, "cross-Gram workspace allocation failed");
    }
    for (int ch = 0; ch < nch; ch++) {
        const int64_t r0 = (int64_t)ch * prow, r1 = std::min(n, r0 + prow);
        const unsigned g = (unsigned)std::min<int64_t>((int64_t)cwb_num_sms() * 16, ((r1 - r0) * ld + 255) / 256);
        if (c->idx_bytes == 1)
            k_gram_P<uint8_t><<<g, 256, 0, s>>>((const uint8_t*)c->idx, n, r0, r1, K, ns, d, ld, c->zj0, c->Zs, P);
        else
            k_gram_P<uint16_t><<<g, 256, 0, s>>>((const uint16_t*)c->idx, n, r0, r1, K, ns, d, ld, c->zj0, c->Zs, P);
        c->launches++;
        // U_k[l][.] = sum over bin l of P rows (k' >= k); the kernels index rows globally: P's base shifted by r0
        const double* Pv = P - r0 * (int64_t)ld;
        if (CR > 0) h1_chunk(c, Pv, ld, K, ns, c->perm, c->perm_bytes, U, nch, ch, s, d);
        else h1(c, Pv, ld, K, ns, c->off, c->perm, c->perm_bytes, U, s, d);
    }
    k_h234<<<dim3(K, ld / 32), 256, 0, s>>>(U, ld, ns, d, c->ZT, c->W, c->lwin, c->Ainv, c->G, nullptr, nullptr,
                                             nullptr, nullptr, nullptr, 0, xg, 1);  // projection Zb_k^T U_k
    k_gram_sym<<<K * d, 256, 0, s>>>(xg, K, d, ld);
    k_gram_w<<<K * d, 256, 0, s>>>(xg, c->Ainv, K, d, ld, Wt);
    c->launches += 3;
    cwb_release(P, s);
    cwb_release(U, s);
    cwb_release(xg, s);
    c->xg = Wt;
    c->xg_ld = ld;
    return cwb_check_launch(c, "cross-Gram kernels");
}

int cwb_train_gram(cwb_ctx* c, const double* Y, int32_t B, double nu, int32_t M, double* offset_out,
                   double* theta_agg_out, int32_t* k_trace, double* sse_trace, double* risk_trace, cudaStream_t s) {
    const int K = c->K, d = c->d;
    {   // k_gram_train keeps theta of every learner (K d doubles) and delta (K) of its replication in shared memory
        int dev = 0, optin = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        if (sizeof(double) * ((size_t)K * d + K) + 1024 > (size_t)optin)
            return cwb_set_error(c, CWB_EUNSUPPORTED, "cwb_train (path 3): K d too large for the cross-Gram kernel");
    }
    int rc = gram_build(c, s);
    if (rc) return rc;
    rc = ensure_ws(c, B, s);
    if (rc) return rc;
    cwb_train_ws& w = c->ws;
    const int Bp = w.Bp;
    double* off_ws = w.rr + Bp;
    rc = column_stats(c, Y, B, true, off_ws, w.rr, offset_out, s);   // f0 = mean(y), r^T r (Alg. 1 lines 2-4)
    if (rc) return rc;
    dim3 gt((unsigned)((c->n + 31) / 32), Bp / 32);
    k_tr_in<<<gt, dim3(32, 8), 0, s>>>(Y, c->n, B, Bp, off_ws, nullptr, w.Rt);
    // theta^[0] = A^-1 Z^T r^[0]: H1-H3 of the initial residuals (k_h234 also writes delta, unused here)
    h1(c, w.Rt, Bp, K, c->n_star, c->off, c->perm, c->perm_bytes, w.U, s);
    k_h234<<<dim3(K, Bp / 32), 256, 0, s>>>(w.U, Bp, c->n_star, d, c->ZT, c->W, c->lwin, c->Ainv, c->G, w.theta,
                                             w.delta);
    const size_t smem = sizeof(double) * ((size_t)K * d + K);
    CWB_CUDA_TRY(c, cudaFuncSetAttribute(k_gram_train, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_gram_train<<<B, 256, smem, s>>>(w.theta, Bp, w.rr, c->xg, c->xg_ld, c->Cb, c->G, K, d, c->n, nu, M, B,
                                       theta_agg_out, k_trace, sse_trace, risk_trace);
    c->launches += 4;
    return cwb_check_launch(c, "cross-Gram train kernels");
}
