// cwb_fused.cu -- the whole CWB loop (Alg. 1 supp.) for RB = 1 or
// 2 replications per CTA, all M iterations in one launch.
//
// Replications are independent boosting runs that share the binned pool, so
// a CTA never waits for another CTA: no grid barrier, no atomics, no host
// round trip between iterations.  The residuals r (n x RB doubles, the RB
// replications of a row side by side) and the bin sums u (K x n* x RB) stay
// in shared memory for all M iterations; when it fits, the read-only pool
// tables used every iteration (gather schedule, basis windows, cached
// inverses, selection factors) are staged in shared memory too, otherwise
// they are read through L1/L2.  Four block barriers per iteration m:
//
//   A  H1  u_k(l) = sum_{i in bin l of learner k} r_i      binMatVec loop
//          The K*n* bins are cut into tasks, sorted by length and dealt to the
//          T threads in snake order by a plan built once per (data set, RB, T)
//          (k_fused_plan).  For each warp the plan holds a gather schedule of
//          byte offsets ([step/4][lane][4]) in which the lanes of a shared-
//          memory wavefront always hit distinct bank groups; one 8- or 16-byte
//          load fetches 4 offsets and each offset addresses the RB residuals of
//          a row directly.  Zero padding rows r[n..n+15] absorb ragged ends; a
//          bin cut into several tasks is completed by a fixed-order combine.
//   B  H2-H4  one warp per learner, lane j = coefficient j:
//          s = Zb^T u over the design-point window of basis j,
//          theta = (G + lambda D)^-1 s with the cached inverse,
//          delta = |C^T theta|^2 = 2 theta^T s - theta^T G theta with C C^T = G + 2 lambda D
//          banded, so SSE_k = r^T r - delta_k.
//   C  H5  warp q (replication q): k* = argmax delta_k, lowest k on ties;
//          zhat = nu Zb_k* theta_k* at the design points; theta_agg[k*] += nu theta* (P:L838).
//   D  H6  r_i -= zhat[idx_k*(i)], r^T r per warp.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <mutex>
#include <vector>

#include "cwb_internal.cuh"

namespace {

constexpr int kDiscard = INT32_MIN;
constexpr int kAregD = 24;  // basis dimension of the register-resident A^-1 columns (the default d)
constexpr int kPadRows = 16;  // zero rows after the n residual rows, one per bank group
constexpr int kSlackEntries = 256;  // schedule entries after the last block (2 groups of 4 x 32 lanes)

struct FusedParams {
    int n, K, ns, nsp, d, M, B, n_multi, W;
    int permt_cap;  // entries of permt staged in shared memory (POOL)
    int ztab;       // bit 0: Zs / zj0 staged in shared memory, bit 1: the index vectors too
    double nu;
    double gamma;  // ACC: momentum parameter (Alg. 2)
    double inv2n;  // 1 / (2n): risk = r^T r / (2n) without a division on the critical path
    const double* Y;
    const void* idx;
    const void* permt;
    const int32_t* plan;
    const int32_t* zj0;
    const double* Zs;
    const double* ZT;     // K x W x d  basis windows
    const int32_t* lwin;  // K x d x 2  window starts
    const double* Ainv;   // K x d x d
    const double* Cb;     // K x d x 4
    double* offset_out;
    double* agg_out;
    double* agg2_out;    // ACC: theta_h
    int32_t* kcor_trace; // ACC
    int32_t* k_trace;
    double* sse_trace;
    double* risk_trace;
    long long* timing;  // optional: cycles per phase (CTA 0, thread 0), summed over iterations
    int* status;
    // HC (hybrid CWB, Alg. 3): validation mask, training-row tables, patience, extra outputs
    const uint8_t* vmask;  // n, 1 = validation row
    const double* Ainv_tr;  // K x d x d  (G_tr + lambda D)^-1
    const double* Cb_tr;    // K x d x 4  band of C_tr, C_tr C_tr^T = G_tr + 2 lambda D
    int pat0;
    double* val_risk_trace;
    int32_t* switch_iter;
};

__host__ __device__ __forceinline__ size_t align16(size_t b) { return (b + 15) & ~(size_t)15; }

struct SmemLayout {
    size_t r, U, delta, th, ss, zhat, agg, pc, red, permt, zt, ai, cb, lw, zs, zj, ix, total;
    size_t hh;  // ACC: H = y - h (momentum model), n doubles
    size_t ff, mk;  // HC: F = y - f (primary model, all rows), n doubles; validation mask, n bytes
    size_t by, bf;  // BERN: targets y and fit f, n x RB doubles each
    __host__ __device__ SmemLayout(int n, int K, int nsp, int d, int W, int n_multi, int RB, int NW, bool pool,
                                   size_t permt_bytes, int ztab, int idx_bytes = 1, bool acc = false,
                                   bool hc = false, bool bern = false) {
        size_t o = 0;
        r = o; o = align16(o + sizeof(double) * RB * (size_t)(n + kPadRows));  // r[n..n+15] = 0: padding rows
        U = o; o = align16(o + sizeof(double) * RB * ((size_t)K * nsp + W));  // +W: window overrun pad
        delta = o; o = align16(o + sizeof(double) * RB * K);
        th = o; o = align16(o + sizeof(double) * RB * (size_t)K * 32);        // theta_k of every learner
        ss = o; o = align16(o + sizeof(double) * RB * (size_t)NW * 32);       // per-warp s = Zb^T u
        zhat = o; o = align16(o + sizeof(double) * RB * (size_t)nsp);
        agg = o; o = align16(o + sizeof(double) * RB * (size_t)K * d);
        pc = o; o = align16(o + sizeof(double) * RB * (n_multi > 0 ? n_multi : 1));
        red = o; o = align16(o + sizeof(double) * 2 * (RB + (acc ? 1 : 0) + (hc ? 1 : 0) + (bern ? RB : 0)) *
                                 (size_t)NW * 32);
        hh = o; if (acc) o = align16(o + sizeof(double) * (size_t)n);
        ff = o; if (hc) o = align16(o + sizeof(double) * (size_t)n);
        mk = o; if (hc) o = align16(o + (size_t)n);
        by = o; if (bern) o = align16(o + sizeof(double) * RB * (size_t)n);
        bf = o; if (bern) o = align16(o + sizeof(double) * RB * (size_t)n);
        permt = o; if (pool) o = align16(o + permt_bytes);
        zt = o; if (pool) o = align16(o + sizeof(double) * (size_t)K * W * d);
        ai = o; if (pool) o = align16(o + sizeof(double) * (size_t)K * d * d);
        cb = o; if (pool) o = align16(o + sizeof(double) * (size_t)K * d * 4);
        lw = o; if (pool) o = align16(o + sizeof(int32_t) * (size_t)K * d);
        zs = o; if (ztab) o = align16(o + sizeof(double) * (size_t)K * nsp * CWB_SPW);
        zj = o; if (ztab) o = align16(o + sizeof(int32_t) * (size_t)K * nsp);
        ix = o; if (ztab & 2) o = align16(o + (size_t)idx_bytes * K * n);
        total = o;
    }
};

// plan layout (int32), built by k_fused_plan:
//   [0] n_tasks [1] rounds [2] n_comb [3] n_multi [4] P [5] permt entries [6..7] 0
//   tt_dest[R*T]   destination of thread t's task in round r (>= 0: u index,
//                  < 0: piece slot -dest-1, INT32_MIN: no task)
//   wl[R*NW]       steps of warp w in round r (multiple of 8, 0: none)
//   wb[R*NW]       offset of that block in permt ([step/4][lane][4] byte offsets)
//   comb_g[KS] comb_first[KS] comb_cnt[KS]   bins cut into several pieces
__host__ __device__ __forceinline__ int plan_rounds_max(int KS, int T) { return (KS + 2 * T) / T + 1; }
__host__ __device__ __forceinline__ size_t plan_ints(int KS, int T) {
    const size_t R = plan_rounds_max(KS, T);
    return 8 + R * T + 2 * R * (T / 32) + 3 * (size_t)KS;
}
// task cut: bins longer than piece_factor() x the mean bin size are cut into pieces.  Any cut bin costs the
// combine pass and its barrier in every iteration, which outweighs the shorter critical task: R1 (B = 256) per
// iteration 9,565 cycles at 1.6 vs 9,073 at 4.0 (CWB; ACWB 10,900 -> 9,975, HCWB 24,832 -> 23,155, Bernoulli
// 16,027 -> 15,401; profiles/r2h_piece_factor.txt).  4x still cuts outlier bins (heavy ties).  CWB_PFAC
// overrides it for experiments.
static double piece_factor() {
    static const double f = getenv("CWB_PFAC") ? atof(getenv("CWB_PFAC")) : 4.0;
    return f;
}
__host__ __device__ __forceinline__ size_t permt_bound(int KS, int T, int P) {
    return (size_t)plan_rounds_max(KS, T) * T * (size_t)((P + 3) / 4 * 4);
}

template <int RB> struct RV;  // RB residuals of one row
template <> struct RV<1> {
    double x;
    __device__ __forceinline__ static RV ld(const unsigned char* base, uint32_t off) {
        RV v; v.x = *reinterpret_cast<const double*>(base + off); return v;
    }
    __device__ __forceinline__ double operator[](int) const { return x; }
};
template <> struct RV<2> {
    double x, y;
    __device__ __forceinline__ static RV ld(const unsigned char* base, uint32_t off) {
        const double2 t = *reinterpret_cast<const double2*>(base + off); RV v; v.x = t.x; v.y = t.y; return v;
    }
    __device__ __forceinline__ double operator[](int q) const { return q ? y : x; }
};

// 4 byte offsets of consecutive steps of this lane
template <typename PermT> struct Off4;
template <> struct Off4<uint16_t> {
    uint32_t o0, o1, o2, o3;
    template <bool SM> __device__ __forceinline__ static Off4 ld(const uint16_t* p) {
        const uint2 v = SM ? *reinterpret_cast<const uint2*>(p) : __ldg(reinterpret_cast<const uint2*>(p));
        Off4 o; o.o0 = v.x & 0xffffu; o.o1 = v.x >> 16; o.o2 = v.y & 0xffffu; o.o3 = v.y >> 16; return o;
    }
};
template <> struct Off4<uint32_t> {
    uint32_t o0, o1, o2, o3;
    template <bool SM> __device__ __forceinline__ static Off4 ld(const uint32_t* p) {
        const uint4 v = SM ? *reinterpret_cast<const uint4*>(p) : __ldg(reinterpret_cast<const uint4*>(p));
        Off4 o; o.o0 = v.x; o.o1 = v.y; o.o2 = v.z; o.o3 = v.w; return o;
    }
};

template <bool SM> __device__ __forceinline__ double2 ld2(const double2* p) { return SM ? *p : __ldg(p); }

__device__ __forceinline__ long long phase_mark(long long* acc, long long t0, bool on) {
    if (!on) return 0;
    const long long t = clock64();
    *acc += t - t0;
    return t;
}

// ACC (accelerated CWB, Alg. 2): RB = 2 columns of ONE replication per CTA, column 0 the pseudo
// residuals r = y - g, column 1 the error-corrected residuals c; H = y - h in shared memory.
// HC (hybrid CWB, Alg. 3, with ACC): per replication (CTA) ACWB on the training rows while the
// validation-risk patience counter is below pat0, then CWB on all rows from the primary model;
// F = y - f in shared memory, fitting columns zero on validation rows while accelerated, the
// training-row tables (A_tr^-1, C_tr) until the switch, the pool's afterwards.
// BERN (CWB with the Bernoulli loss, NEXT-4): y and f of the RB replications in shared memory,
// offset logit(mean y), pseudo residuals r = y - sigma(f), risk = mean log-loss.
template <typename IdxT, typename PermT, int RB, bool POOL, int MAXT, int MINB, bool ACC = false, bool HC = false,
          bool BERN = false>
__global__ void __launch_bounds__(MAXT, MINB) k_train_fused(FusedParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int T = blockDim.x, NW = T >> 5;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    static_assert(!ACC || RB == 2, "ACWB runs its two columns as RB = 2");
    static_assert(!HC || ACC, "HCWB builds on the ACWB layout");
    static_assert(!BERN || !ACC, "Bernoulli loss: CWB layout");
    const int b0 = ACC ? blockIdx.x : blockIdx.x * RB;  // ACC: the replication; else the first of RB
    const int n = p.n;
    const int K = p.K, ns = p.ns, nsp = p.nsp, d = p.d, KS = K * ns;
    const int W = p.W;
    const SmemLayout L(n, K, nsp, d, W, p.n_multi, RB, NW, POOL, sizeof(PermT) * (size_t)p.permt_cap, p.ztab,
                       (int)sizeof(IdxT), ACC, HC, BERN);
    double* Yb = (double*)(smem + L.by);  // BERN only: Yb[i * RB + q]
    double* Fb = (double*)(smem + L.bf);  // BERN only
    double* Hm = (double*)(smem + L.hh);  // ACC only
    double* Fm = (double*)(smem + L.ff);  // HC only
    uint8_t* mk = (uint8_t*)(smem + L.mk);  // HC only
    double* r = (double*)(smem + L.r);  // r[i * RB + q]
    const unsigned char* rb = smem + L.r;
    double* U = (double*)(smem + L.U);  // U[g * RB + q], g = k * nsp + l
    double* delta = (double*)(smem + L.delta);
    double* thall = (double*)(smem + L.th);  // thall[(k * RB + q) * 32 + j]
    double* zhat = (double*)(smem + L.zhat);  // zhat[q * nsp + l]
    double* agg = (double*)(smem + L.agg);
    double* pc = (double*)(smem + L.pc);
    double* red = (double*)(smem + L.red);  // red[(parity * RB + q) * T + tid]: per-thread r^T r partials
    const PermT* permt = POOL ? (const PermT*)(smem + L.permt) : (const PermT*)p.permt;
    const double* ZTc = POOL ? (const double*)(smem + L.zt) : p.ZT;
    // HC: training-row tables until the switch (POOL: the shared-memory copy is restaged then)
    const double* Ac = POOL ? (const double*)(smem + L.ai) : (HC ? p.Ainv_tr : p.Ainv);
    const double* Cbc = POOL ? (const double*)(smem + L.cb) : (HC ? p.Cb_tr : p.Cb);
    double* sS = (double*)(smem + L.ss) + (size_t)warp * RB * 32;
    // POOL: every per-iteration table is in shared memory (compile-time known: LDS, not generic loads)
    const double* Zs_c = POOL ? (const double*)(smem + L.zs) : p.Zs;
    const int32_t* zj0_c = POOL ? (const int32_t*)(smem + L.zj) : p.zj0;
    const int zstride = POOL ? nsp : ns;  // row stride of Zs / zj0 per learner
    const IdxT* idx = POOL ? (const IdxT*)(smem + L.ix) : (const IdxT*)p.idx;
    const bool timed = p.timing && blockIdx.x == 0 && tid == 0;
    long long tA = 0, tB = 0, tC = 0, tD = 0, tm = 0;
    __shared__ int ks_sh[2];
    __shared__ double best_sh[2];
    __shared__ int hc_ph, hc_pu, hc_pat, hc_sw;  // HC: phase (0 ACWB, 1 CWB), phase of the last fit, counter, switch
    __shared__ double hc_vprev, hc_ntr, hc_nval;

    // ---- prologue: pool staging, plan tables, I8 offset f0 = mean(y) --------
    if (POOL) {
        const uint4* src = (const uint4*)p.permt;
        uint4* dst = (uint4*)(smem + L.permt);
        const int nv = (int)((sizeof(PermT) * (size_t)p.permt_cap) / 16);
        for (int a = tid; a < nv; a += T) dst[a] = __ldg(src + a);
        for (int a = tid; a < K * W * d; a += T) ((double*)(smem + L.zt))[a] = __ldg(p.ZT + a);
        const double* ai_src = HC ? p.Ainv_tr : p.Ainv;
        const double* cb_src = HC ? p.Cb_tr : p.Cb;
        for (int a = tid; a < K * d * d; a += T) ((double*)(smem + L.ai))[a] = __ldg(ai_src + a);
        for (int a = tid; a < K * d * 4; a += T) ((double*)(smem + L.cb))[a] = __ldg(cb_src + a);
        for (int a = tid; a < K * d; a += T) ((int32_t*)(smem + L.lw))[a] = __ldg(p.lwin + 2 * a);
    }
    if (POOL) {
        double* zd = (double*)(smem + L.zs);
        int32_t* jd = (int32_t*)(smem + L.zj);
        for (int a = tid; a < K * ns; a += T) {
            const int k = a / ns, l = a - k * ns;
#pragma unroll
            for (int q = 0; q < CWB_SPW; q++) zd[((size_t)k * nsp + l) * CWB_SPW + q] = __ldg(p.Zs + (size_t)a * CWB_SPW + q);
            jd[k * nsp + l] = __ldg(p.zj0 + a);
        }
    }
    if (POOL) {  // index vectors (K x n), 16-byte copies + tail
        const size_t nb = sizeof(IdxT) * (size_t)K * n, nv = nb / 16;
        const uint4* src = (const uint4*)p.idx;
        uint4* dst = (uint4*)(smem + L.ix);
        for (size_t a = tid; a < nv; a += T) dst[a] = __ldg(src + a);
        for (size_t a = nv * 16 + tid; a < nb; a += T) (smem + L.ix)[a] = ((const unsigned char*)p.idx)[a];
    }
    const int32_t* pl = p.plan;
    const int rounds = pl[1], n_comb = pl[2];
    const int RM = plan_rounds_max(KS, T);
    const int32_t* tt_dest = pl + 8;
    const int32_t* wl = tt_dest + RM * T;
    const int32_t* wb = wl + RM * NW;
    const int32_t* comb_g = wb + RM * NW;
    const int32_t* comb_first = comb_g + KS;
    const int32_t* comb_cnt = comb_first + KS;
    for (int a = tid; a < RB * (K * nsp + W); a += T) U[a] = 0.0;  // empty / padding bins keep u = 0
    for (int a = tid; a < RB * K * d; a += T) agg[a] = 0.0;
    for (int a = tid; a < RB * kPadRows; a += T) r[n * RB + a] = 0.0;

    // per-thread partial slots: r^T r of the RB columns (+ F^2 for ACC, + F^2 on D_val for HC,
    // + the log-loss of the RB columns for BERN)
    const int NRB = RB + (ACC ? 1 : 0) + (HC ? 1 : 0) + (BERN ? RB : 0);
    double f0[RB];
    if (HC) {
        // f0 = mean of the training targets (Alg. 3 / Alg. 2 line 2 on D_train); F = H = y - f0 on all
        // rows; fitting columns r = c = y - f0 on the training rows, 0 on the validation rows;
        // r^T r over the training rows; validation risk of f0 = sum_val (y - f0)^2 / (2 n_val)
        double sy = 0.0, ntr = 0.0;
        bool bad = false;
        for (int i = tid; i < n; i += T) {
            const uint8_t v_ = p.vmask[i];
            mk[i] = v_;
            const double y = p.Y[(size_t)b0 * n + i];
            bad |= !isfinite(y);
            Fm[i] = y;
            if (!v_) { sy += y; ntr += 1.0; }
        }
        if (bad) cwb_dev_fail(p.status, CWB_ENONFINITE);
        sy = warp_sum(sy);
        ntr = warp_sum(ntr);
        if (lane == 0) { red[warp] = sy; red[32 + warp] = ntr; }
        __syncthreads();
        double st = 0.0, nt = 0.0;
        for (int w = 0; w < NW; w++) { st += red[w]; nt += red[32 + w]; }
        f0[0] = f0[RB - 1] = st / nt;
        double ptr = 0.0, pv = 0.0;
        for (int i = tid; i < n; i += T) {
            const double v = Fm[i] - f0[0];
            Fm[i] = v;
            Hm[i] = v;
            const double vm = mk[i] ? 0.0 : v;
            r[2 * i] = vm;
            r[2 * i + 1] = vm;
            ptr += vm * vm;
            if (mk[i]) pv += v * v;
        }
        __syncthreads();  // everyone has read red[] for f0
        red[(NRB + 0) * T + tid] = ptr;  // rr_0 of both columns -> parity 1
        red[(NRB + 1) * T + tid] = ptr;
        pv = warp_sum(pv);
        __shared__ double s_pv[32];
        if (lane == 0) s_pv[warp] = pv;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < NW; w++) t += s_pv[w];
            hc_ntr = nt;
            hc_nval = (double)n - nt;
            hc_vprev = t / (2.0 * hc_nval);
            hc_ph = 0;
            hc_pu = 0;
            hc_pat = 0;
            hc_sw = p.M;
        }
        __syncthreads();
    } else if (BERN) {
        // Alg. 1 line 2 with the Bernoulli loss: f0 = logit(mean y), y in {0, 1};
        // r = y - sigma(f0) (line 4); r^T r
        double part[RB];
        bool bad = false, nb01 = false;
#pragma unroll
        for (int q = 0; q < RB; q++) part[q] = 0.0;
        for (int i = tid; i < n; i += T) {
#pragma unroll
            for (int q = 0; q < RB; q++) {
                const int bq = b0 + q;
                const double v = (bq < p.B) ? p.Y[(size_t)bq * n + i] : (double)(i & 1);  // padding column
                bad |= !isfinite(v);
                nb01 |= v != 0.0 && v != 1.0;
                Yb[i * RB + q] = v;
                part[q] += v;
            }
        }
        if (bad) cwb_dev_fail(p.status, CWB_ENONFINITE);
        if (nb01) cwb_dev_fail(p.status, CWB_EINVAL);
#pragma unroll
        for (int q = 0; q < RB; q++) {
            part[q] = warp_sum(part[q]);
            if (lane == 0) red[q * 32 + warp] = part[q];
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < RB; q++) {
            double sy = 0.0;
            for (int w = 0; w < NW; w++) sy += red[q * 32 + w];
            const double pb = sy / (double)n;
            if (!(pb > 0.0 && pb < 1.0) && b0 + q < p.B && tid == 0) cwb_dev_fail(p.status, CWB_EDEGENERATE);
            f0[q] = log(pb / (1.0 - pb));
            part[q] = 0.0;
        }
        for (int i = tid; i < n; i += T) {
#pragma unroll
            for (int q = 0; q < RB; q++) {
                const double f = f0[q];
                double lo;
                const double v = bern_resid(Yb[i * RB + q], f, &lo);
                Fb[i * RB + q] = f;
                r[i * RB + q] = v;
                part[q] += v * v;
            }
        }
        __syncthreads();  // everyone has read red[] for f0
#pragma unroll
        for (int q = 0; q < RB; q++) red[(NRB + q) * T + tid] = part[q];  // rr_0 -> parity 1
        __syncthreads();
    } else {
        double part[RB];
        bool bad = false;
#pragma unroll
        for (int q = 0; q < RB; q++) part[q] = 0.0;
        for (int i = tid; i < n; i += T) {
#pragma unroll
            for (int q = 0; q < RB; q++) {
                const int bq = ACC ? b0 : b0 + q;
                const double v = (bq < p.B) ? p.Y[(size_t)bq * n + i] : 0.0;
                bad |= !isfinite(v);
                r[i * RB + q] = v;
                part[q] += v;
            }
        }
        if (bad) cwb_dev_fail(p.status, CWB_ENONFINITE);
#pragma unroll
        for (int q = 0; q < RB; q++) {
            part[q] = warp_sum(part[q]);
            if (lane == 0) red[q * 32 + warp] = part[q];
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < RB; q++) {
            double sy = 0.0;
            for (int w = 0; w < NW; w++) sy += red[q * 32 + w];
            f0[q] = sy / (double)n;
            part[q] = 0.0;
        }
        for (int i = tid; i < n; i += T) {
#pragma unroll
            for (int q = 0; q < RB; q++) {
                const double v = r[i * RB + q] - f0[q];
                r[i * RB + q] = v;
                part[q] += v * v;
            }
        }
        __syncthreads();  // everyone has read red[] for f0
#pragma unroll
        for (int q = 0; q < RB; q++) red[(NRB + q) * T + tid] = part[q];  // rr_0 -> parity 1
        if (ACC)  // f = h = g = f0 (Alg. 2 line 2): H = y - f0; r = c = y - f0 already
            for (int i = tid; i < n; i += T) Hm[i] = r[i * RB];
        __syncthreads();
    }
    if (timed) tm = clock64();

    // Bookkeeping of iteration mp for replication q (one warp): theta_agg[k*] += nu theta*
    // (P:L838), traces k*, SSE = rr_mp - delta* and risk = rr_(mp+1) / (2n), with rr_m the
    // per-thread partials of r^T r before the update of iteration m (parity (m+1) & 1).
    // Runs in phase A of iteration mp + 1 on the first warps (least H1 work, lowest issue
    // priority), off the critical path.
    auto bookkeeping_acc = [&](int mp) {
        // Alg. 2 parameters: theta_g = (1-vt) theta_f + vt theta_h; theta_f = theta_g + nu e_k theta;
        // theta_h += eta e_kcor theta_cor; traces; risk of f = F^T F / (2n) (slot RB, parity mp)
        const double vt = 2.0 / (double)(mp + 2), eta = p.gamma * p.nu / vt;
        const int k0 = ks_sh[0], k1 = ks_sh[1];
        double* tf = agg;
        double* th = agg + K * d;
        for (int a = lane; a < K * d; a += 32) tf[a] = (1.0 - vt) * tf[a] + vt * th[a];
        __syncwarp();
        if (lane < d) {
            tf[k0 * d + lane] += p.nu * thall[(k0 * RB + 0) * 32 + lane];
            th[k1 * d + lane] += eta * thall[(k1 * RB + 1) * 32 + lane];
        }
        double s0 = 0.0, sf = 0.0;
        for (int t = lane; t < T; t += 32) {
            s0 += red[((mp + 1) & 1) * NRB * T + t];
            sf += red[(mp & 1) * NRB * T + RB * T + t];
        }
        const double rr0 = warp_sum(s0), rf = warp_sum(sf);
        if (lane == 0 && b0 < p.B) {
            if (p.k_trace) p.k_trace[(size_t)mp * p.B + b0] = k0;
            if (p.kcor_trace) p.kcor_trace[(size_t)mp * p.B + b0] = k1;
            if (p.sse_trace) p.sse_trace[(size_t)mp * p.B + b0] = rr0 - best_sh[0];
            if (p.risk_trace) p.risk_trace[(size_t)mp * p.B + b0] = rf * p.inv2n;
        }
    };
    auto bookkeeping_hc = [&](int mp) {
        // Alg. 3: the fit of iteration mp ran in phase hc_pu: 0 -> ACWB bookkeeping of theta_f,
        // theta_h; 1 -> CWB aggregation theta_f[k] += nu theta.  Traces k, kcor (-1 after the
        // switch), SSE = rr_mp - delta*; the risk traces are written by the decide step.
        const double vt = 2.0 / (double)(mp + 2), eta = p.gamma * p.nu / vt;
        const int k0 = ks_sh[0], k1 = ks_sh[1];
        const bool accel = hc_pu == 0;
        double* tf = agg;
        double* th = agg + K * d;
        if (accel) {
            for (int a = lane; a < K * d; a += 32) tf[a] = (1.0 - vt) * tf[a] + vt * th[a];
            __syncwarp();
        }
        if (lane < d) {
            tf[k0 * d + lane] += p.nu * thall[(k0 * RB + 0) * 32 + lane];
            if (accel) th[k1 * d + lane] += eta * thall[(k1 * RB + 1) * 32 + lane];
        }
        double s0 = 0.0;
        for (int t = lane; t < T; t += 32) s0 += red[((mp + 1) & 1) * NRB * T + t];
        const double rr0 = warp_sum(s0);
        if (lane == 0 && b0 < p.B) {
            if (p.k_trace) p.k_trace[(size_t)mp * p.B + b0] = k0;
            if (p.kcor_trace) p.kcor_trace[(size_t)mp * p.B + b0] = accel ? k1 : -1;
            if (p.sse_trace) p.sse_trace[(size_t)mp * p.B + b0] = rr0 - best_sh[0];
        }
    };
    auto bookkeeping = [&](int mp, int q) {
        const int b = b0 + q, kb = ks_sh[q];
        if (lane < d) agg[(q * K + kb) * d + lane] += p.nu * thall[(kb * RB + q) * 32 + lane];
        double s0 = 0.0, s1 = 0.0;
        for (int t = lane; t < T; t += 32) {
            s0 += red[((mp + 1) & 1) * NRB * T + q * T + t];
            s1 += red[(mp & 1) * NRB * T + ((BERN ? RB : 0) + q) * T + t];  // BERN: the log-loss slot
        }
        const double rr0 = warp_sum(s0), rr1 = warp_sum(s1);
        if (lane == 0 && b < p.B) {
            if (p.k_trace) p.k_trace[(size_t)mp * p.B + b] = kb;
            if (p.sse_trace) p.sse_trace[(size_t)mp * p.B + b] = rr0 - best_sh[q];
            if (p.risk_trace) p.risk_trace[(size_t)mp * p.B + b] = BERN ? rr1 * (2.0 * p.inv2n) : rr1 * p.inv2n;
        }
    };

    // CWB with two replications per 384-thread CTA (register budget 170): when every learner has its own warp
    // and d = 24, lane j of learner k's warp keeps column j of A_k^-1 in registers for phase B (the per-iteration
    // A^-1 stream from shared memory was phase B's bound at R1)
    constexpr bool AREG_T = (MAXT == 384 && RB == 2 && !ACC && !HC && !BERN);
    const bool areg = AREG_T && K <= NW && d == kAregD;
    double Areg[AREG_T ? kAregD : 1];
#pragma unroll
    for (int jp = 0; jp < (AREG_T ? kAregD : 1); jp++)
        Areg[jp] = (AREG_T && areg && warp < K && lane < d) ? Ac[((size_t)warp * d + jp) * d + lane] : 0.0;

    for (int m = 0; m < p.M; m++) {
        if (HC) {
            if (m > 0 && warp == 0) bookkeeping_hc(m - 1);
        } else if (ACC) {
            if (m > 0 && warp == 0) bookkeeping_acc(m - 1);
        } else if (m > 0 && warp < RB) {
            bookkeeping(m - 1, warp);
        }
        CWB_JIT(m * 8 + 0);
        // ---- A / H1: each lane sums its task, 4 steps per offset load ------------------
        for (int rd = 0; rd < rounds; rd++) {
            const int steps = __ldg(wl + rd * NW + warp);  // warp-uniform
            if (steps == 0) continue;
            const PermT* pt = permt + __ldg(wb + rd * NW + warp) + lane * 4;
            double a0[RB], a1[RB];
#pragma unroll
            for (int q = 0; q < RB; q++) { a0[q] = 0.0; a1[q] = 0.0; }
            // software pipeline: the offsets of groups g+2, g+3 load while groups g, g+1 gather
            // (steps are a multiple of 8; the schedule buffer has 2 groups of slack at its end)
            const int ng = steps >> 2;  // groups of 4 steps, even
            Off4<PermT> oa = Off4<PermT>::template ld<POOL>(pt);
            Off4<PermT> ob = Off4<PermT>::template ld<POOL>(pt + 128);
            for (int g = 0; g < ng; g += 2) {
                const Off4<PermT> na = Off4<PermT>::template ld<POOL>(pt + (g + 2) * 128);
                const Off4<PermT> nb = Off4<PermT>::template ld<POOL>(pt + (g + 3) * 128);
                const RV<RB> v0 = RV<RB>::ld(rb, oa.o0), v1 = RV<RB>::ld(rb, oa.o1);
                const RV<RB> v2 = RV<RB>::ld(rb, oa.o2), v3 = RV<RB>::ld(rb, oa.o3);
                const RV<RB> v4 = RV<RB>::ld(rb, ob.o0), v5 = RV<RB>::ld(rb, ob.o1);
                const RV<RB> v6 = RV<RB>::ld(rb, ob.o2), v7 = RV<RB>::ld(rb, ob.o3);
#pragma unroll
                for (int q = 0; q < RB; q++) {
                    a0[q] += v0[q]; a1[q] += v1[q]; a0[q] += v2[q]; a1[q] += v3[q];
                    a0[q] += v4[q]; a1[q] += v5[q]; a0[q] += v6[q]; a1[q] += v7[q];
                }
                oa = na;
                ob = nb;
            }
            const int dest = __ldg(tt_dest + rd * T + tid);
            double* dp = dest >= 0 ? U + (size_t)dest * RB : (dest != kDiscard ? pc + (size_t)(-dest - 1) * RB : nullptr);
            if (dp) {
                if (RB == 2) *reinterpret_cast<double2*>(dp) = make_double2(a0[0] + a1[0], a0[RB - 1] + a1[RB - 1]);
                else dp[0] = a0[0] + a1[0];
            }
        }
        if (n_comb) {  // bins cut into pieces: combine in piece order
            __syncthreads();
            for (int c = tid; c < n_comb; c += T) {
                const int f = __ldg(comb_first + c), cnt = __ldg(comb_cnt + c), g = __ldg(comb_g + c);
#pragma unroll
                for (int q = 0; q < RB; q++) {
                    double v = pc[f * RB + q];
                    for (int e = 1; e < cnt; e++) v += pc[(f + e) * RB + q];
                    U[g * RB + q] = v;
                }
            }
        }
#ifdef CWB_PHASE_DEBUG
        __shared__ long long dbg_endA[32], dbg_endB[32];
        if (lane == 0) dbg_endA[warp] = clock64();
#endif
        __syncthreads();
        if (timed) tm = phase_mark(&tA, tm, true);
        CWB_JIT(m * 8 + 1);
        // ---- B / H2-H4, one warp per learner, lane j = coefficient j:
        //      s = Zb^T u (window of basis j), theta = (G + lambda D)^-1 s (cached inverse,
        //      P:L846), c = C^T theta, delta = |c|^2 = 2 theta^T s - theta^T G theta ------
        for (int k = warp; k < K; k += NW) {
#ifdef CWB_PHASE_DEBUG
            long long dt0 = 0;
            const bool dbgw = timed || (blockIdx.x == 0 && warp == 0 && lane == 0);
            if (dbgw) { if (__double_as_longlong(U[k * nsp * RB]) == 0x7ff8deadbeefll) dt0 = 1; dt0 += clock64(); }
#endif
            double sv[RB];
#pragma unroll
            for (int q = 0; q < RB; q++) sv[q] = 0.0;
            __syncwarp();  // sS reuse
            if (lane < d) {
                const double* zt = ZTc + (size_t)k * W * d + lane;
                const int lb = POOL ? ((const int32_t*)(smem + L.lw))[k * d + lane] : __ldg(p.lwin + 2 * (k * d + lane));
                const double* uk = U + ((size_t)k * nsp + lb) * RB;
#pragma unroll 4
                for (int w = 0; w < W; w++) {
                    const double z = POOL ? zt[w * d] : __ldg(zt + w * d);
                    if (RB == 2) {
                        const double2 u2 = *reinterpret_cast<const double2*>(uk + 2 * w);
                        sv[0] = fma(z, u2.x, sv[0]);
                        sv[RB - 1] = fma(z, u2.y, sv[RB - 1]);
                    } else {
                        sv[0] = fma(z, uk[w], sv[0]);
                    }
                }
            }
#ifdef CWB_PHASE_DEBUG
            long long dts = 0;
            if (dbgw) { if (__double_as_longlong(sv[0]) == 0x7ff8deadbeefll) dts = 1; dts += clock64(); }
#endif
#pragma unroll
            for (int q = 0; q < RB; q++) sS[q * 32 + lane] = sv[q];  // lanes >= d store 0
            __syncwarp();
            double t0[RB], t1[RB];
#pragma unroll
            for (int q = 0; q < RB; q++) { t0[q] = 0.0; t1[q] = 0.0; }
            if (AREG_T && areg) {
                if (lane < d) {  // same products and order as the loop below (even jp -> t0, odd -> t1)
#pragma unroll
                    for (int jp = 0; jp < (AREG_T ? kAregD : 2); jp += 2) {
#pragma unroll
                        for (int q = 0; q < RB; q++) {
                            const double2 s2 = *reinterpret_cast<const double2*>(sS + q * 32 + jp);
                            t0[q] = fma(Areg[jp], s2.x, t0[q]);
                            t1[q] = fma(Areg[jp + 1], s2.y, t1[q]);
                        }
                    }
                }
            } else if (lane < d) {
                const double* Ak = Ac + (size_t)k * d * d + lane;  // A^-1 symmetric: column j = row j
                int jp = 0;
#pragma unroll 4
                for (; jp + 2 <= d; jp += 2) {
                    const double a0 = POOL ? Ak[jp * d] : __ldg(Ak + jp * d);
                    const double a1 = POOL ? Ak[(jp + 1) * d] : __ldg(Ak + (jp + 1) * d);
#pragma unroll
                    for (int q = 0; q < RB; q++) {
                        const double2 s2 = *reinterpret_cast<const double2*>(sS + q * 32 + jp);
                        t0[q] = fma(a0, s2.x, t0[q]);
                        t1[q] = fma(a1, s2.y, t1[q]);
                    }
                }
                if (jp < d) {
                    const double a0 = POOL ? Ak[jp * d] : __ldg(Ak + jp * d);
#pragma unroll
                    for (int q = 0; q < RB; q++) t0[q] = fma(a0, sS[q * 32 + jp], t0[q]);
                }
            }
#ifdef CWB_PHASE_DEBUG
            long long dtt = 0;
            if (dbgw) { if (__double_as_longlong(t0[0] + t1[0]) == 0x7ff8deadbeefll) dtt = 1; dtt += clock64(); }
#endif
            double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
            if (lane < d) {
                const double* cbj = Cbc + ((size_t)k * d + lane) * 4;
                c0 = cbj[0]; c1 = cbj[1]; c2 = cbj[2]; c3 = cbj[3];
            }
#pragma unroll
            for (int q = 0; q < RB; q++) {
                const double th = t0[q] + t1[q];  // 0 on lanes >= d
                const double h1 = __shfl_down_sync(0xffffffffu, th, 1);
                const double h2 = __shfl_down_sync(0xffffffffu, th, 2);
                const double h3 = __shfl_down_sync(0xffffffffu, th, 3);
                const double c = fma(c3, h3, fma(c2, h2, fma(c1, h1, c0 * th)));
                const double v = warp_sum(c * c);
                thall[(k * RB + q) * 32 + lane] = th;
                if (lane == 0) delta[k * RB + q] = v;
#ifdef CWB_PHASE_DEBUG
                if (dbgw && q == RB - 1) {
                    long long dte = 0;
                    if (__double_as_longlong(v) == 0x7ff8deadbeefll) dte = 1;
                    dte += clock64();
                    if (timed) { p.timing[60] += dts - dt0; p.timing[61] += dtt - dts; p.timing[62] += dte - dtt; }
                }
#endif
            }
        }
#ifdef CWB_PHASE_DEBUG
        if (lane == 0) dbg_endB[warp] = clock64();
#endif
        __syncthreads();
#ifdef CWB_PHASE_DEBUG
        if (timed) {  // CTA 0: A-phase spread over warps, B after the last A warp, which warp ends A last
            long long mn = dbg_endA[0], mx = dbg_endA[0], mb = dbg_endB[0];
            int wl = 0;
            for (int x = 1; x < NW; x++) {
                mn = min(mn, dbg_endA[x]);
                if (dbg_endA[x] > mx) { mx = dbg_endA[x]; wl = x; }
                mb = max(mb, dbg_endB[x]);
            }
            p.timing[4] += mx - mn;
            p.timing[5] += mb - mx;
            p.timing[8 + wl] += 1;
            for (int x = 0; x < NW; x++) p.timing[40 + x] += dbg_endA[x] - mn;
        }
#endif
        if (timed) tm = phase_mark(&tB, tm, true);
        CWB_JIT(m * 8 + 2);
        // ---- C / H5: job (q, slice): k* = argmax delta (lowest k on ties) for
        //      replication q, then zhat = nu Zb_k* theta_k* on design points slice*32 + lane ------
        {
            const int nslice = (ns + 31) >> 5;
            for (int job = warp; job < RB * nslice; job += NW) {
                const int q = job % RB, sl = job / RB;
                double best = -INFINITY;
                int kb = 0;
                if (K <= 16) {
                    // every lane scans the K deltas in k order (broadcast loads, strict >: the lowest k of
                    // the maximum), the same result as the lane-strided scan + shuffle tree below without
                    // its five dependent shuffle rounds
                    double dv[16];
#pragma unroll
                    for (int k = 0; k < 16; k++) dv[k] = k < K ? delta[k * RB + q] : -INFINITY;
#pragma unroll
                    for (int k = 0; k < 16; k++)
                        if (dv[k] > best) { best = dv[k]; kb = k; }
                } else {
                    for (int k = lane; k < K; k += 32) {
                        const double v = delta[k * RB + q];
                        if (v > best) { best = v; kb = k; }
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                        const int ok = __shfl_xor_sync(0xffffffffu, kb, o);
                        if (ob > best || (ob == best && ok < kb)) { best = ob; kb = ok; }
                    }
                }
                const int l = sl * 32 + lane;
                if (l < ns) {
                    const double* tk = thall + (kb * RB + q) * 32;
                    const int a = zj0_c[(size_t)kb * zstride + l];
                    const double2* zs = reinterpret_cast<const double2*>(Zs_c + ((size_t)kb * zstride + l) * CWB_SPW);
                    const double2 za = zs[0], zb = zs[1];
                    double v = za.x * tk[a];
                    if (a + 1 < d) v += za.y * tk[a + 1];
                    if (a + 2 < d) v += zb.x * tk[a + 2];
                    if (a + 3 < d) v += zb.y * tk[a + 3];
                    zhat[q * nsp + l] = (ACC && q == 1) ? v : p.nu * v;  // ACC: b_kcor unscaled
                }
                if (sl == 0 && lane == 0) { ks_sh[q] = kb; best_sh[q] = best; }
            }
        }
        __syncthreads();
        if (timed) tm = phase_mark(&tC, tm, true);
        CWB_JIT(m * 8 + 3);
        // ---- D / H6: r_i -= zhat[idx_k*(i)], per-thread r^T r partials -------------
        if (HC) {
            // D1: models after iteration m (phase hc_ph): ACWB F = (1-vt) F + vt H - nu b_k (= y - (g + nu b_k)),
            //     H -= eta b_kcor; CWB F -= nu b_k.  Partials of F^2 on all rows and on D_val.
            const int parw = m & 1;
            const bool accel = hc_ph == 0;
            const IdxT* ik0 = idx + (size_t)ks_sh[0] * n;
            const IdxT* ik1 = idx + (size_t)ks_sh[1] * n;
            const double vt = 2.0 / (double)(m + 2), eta = p.gamma * p.nu / vt;
            const double vt1 = 2.0 / (double)(m + 3), a1 = (double)(m + 2) / (double)(m + 3);
            double accA = 0.0, accV = 0.0;
            for (int i = tid; i < n; i += T) {
                const double bk = zhat[ik0[i]];
                const double F = Fm[i];
                double Fn;
                if (accel) {
                    const double Hh = Hm[i];
                    Fn = (1.0 - vt) * F + vt * Hh - bk;
                    Hm[i] = Hh - eta * zhat[nsp + ik1[i]];
                } else {
                    Fn = F - bk;
                }
                Fm[i] = Fn;
                accA = fma(Fn, Fn, accA);
                if (mk[i]) accV = fma(Fn, Fn, accV);
            }
            red[(parw * NRB + RB) * T + tid] = accA;
            red[(parw * NRB + RB + 1) * T + tid] = accV;
            __syncthreads();
            CWB_JIT(m * 8 + 4);
            // decide (Alg. 3 line 6): risk traces, patience counter, one-way switch to CWB
            if (warp == 0) {
                double sa = 0.0, sv = 0.0;
                for (int t = lane; t < T; t += 32) {
                    sa += red[(parw * NRB + RB) * T + t];
                    sv += red[(parw * NRB + RB + 1) * T + t];
                }
                sa = warp_sum(sa);
                sv = warp_sum(sv);
                if (lane == 0) {
                    const double vr = sv / (2.0 * hc_nval);
                    if (b0 < p.B) {
                        if (p.risk_trace) p.risk_trace[(size_t)m * p.B + b0] = sa * p.inv2n;
                        if (p.val_risk_trace) p.val_risk_trace[(size_t)m * p.B + b0] = vr;
                    }
                    hc_pu = hc_ph;
                    if (hc_ph == 0) {
                        hc_pat = vr > hc_vprev ? hc_pat + 1 : 0;
                        if (hc_pat >= p.pat0) {
                            hc_ph = 1;
                            hc_sw = m + 1;
                        }
                    }
                    hc_vprev = vr;
                }
            }
            __syncthreads();
            CWB_JIT(m * 8 + 5);
            const bool accel1 = hc_ph == 0;
            if (accel && !accel1) {  // switched: the pool's tables from now on
                if (POOL) {
                    for (int a = tid; a < K * d * d; a += T) ((double*)(smem + L.ai))[a] = __ldg(p.Ainv + a);
                    for (int a = tid; a < K * d * 4; a += T) ((double*)(smem + L.cb))[a] = __ldg(p.Cb + a);
                } else {
                    Ac = p.Ainv;
                    Cbc = p.Cb;
                }
            }
            // D2: fitting columns of iteration m+1.  ACWB: r' = (1-vt1) F + vt1 H, c' = r' + a1 (c - b_kcor),
            //     zero on D_val; CWB: r' = F on all rows, c' = 0.  Partials of r'^2, c'^2.
            double acc0 = 0.0, acc1 = 0.0;
            for (int i = tid; i < n; i += T) {
                double rn, cn;
                if (accel1) {
                    rn = (1.0 - vt1) * Fm[i] + vt1 * Hm[i];
                    cn = rn + a1 * (r[2 * i + 1] - zhat[nsp + ik1[i]]);
                    if (mk[i]) { rn = 0.0; cn = 0.0; }
                } else {
                    rn = Fm[i];
                    cn = 0.0;
                }
                *reinterpret_cast<double2*>(r + 2 * i) = make_double2(rn, cn);
                acc0 = fma(rn, rn, acc0);
                acc1 = fma(cn, cn, acc1);
            }
            red[(parw * NRB + 0) * T + tid] = acc0;
            red[(parw * NRB + 1) * T + tid] = acc1;
        } else {
            const int parw = m & 1;
            const IdxT* ik0 = idx + (size_t)ks_sh[0] * n;
            const IdxT* ik1 = idx + (size_t)ks_sh[RB - 1] * n;
            double acc[RB], accF = 0.0, accL[RB];
#pragma unroll
            for (int q = 0; q < RB; q++) { acc[q] = 0.0; accL[q] = 0.0; }
            // ACC (Alg. 2, ACWB iteration ma = m + 1): F = r - nu b_k (line 8), H -= eta b_kcor (line 16),
            // next columns r' = (1 - vt1) F + vt1 H (lines 4-6), c' = r' + a1 (c - b_kcor) (line 10)
            const double vt = 2.0 / (double)(m + 2), eta = p.gamma * p.nu / vt;
            const double vt1 = 2.0 / (double)(m + 3), a1 = (double)(m + 2) / (double)(m + 3);
            for (int i0 = tid; i0 < n; i0 += 4 * T) {
                uint32_t j0[4], j1[4];
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    const int i = i0 + e * T;
                    j0[e] = i < n ? (uint32_t)ik0[i] : 0u;
                    j1[e] = (RB == 2 && i < n) ? (uint32_t)ik1[i] : 0u;
                }
                if (!BERN && !ACC) {
                    // plain CWB: the four rows' r and zhat loads are issued before the first store (the
                    // compiler cannot reorder loads past the r stores itself); same arithmetic and order
                    double2 rv[4];
                    double z0[4], z1[4];
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        const int i = i0 + e * T;
                        if (i < n) {
                            if (RB == 1) rv[e].x = r[i];
                            else rv[e] = *reinterpret_cast<const double2*>(r + 2 * i);
                            z0[e] = zhat[j0[e]];
                            z1[e] = RB == 2 ? zhat[nsp + j1[e]] : 0.0;
                        }
                    }
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        const int i = i0 + e * T;
                        if (i < n) {
                            if (RB == 1) {
                                const double v = rv[e].x - z0[e];
                                r[i] = v;
                                acc[0] = fma(v, v, acc[0]);
                            } else {
                                double2 v = rv[e];
                                v.x -= z0[e];
                                v.y -= z1[e];
                                *reinterpret_cast<double2*>(r + 2 * i) = v;
                                acc[0] = fma(v.x, v.x, acc[0]);
                                acc[RB - 1] = fma(v.y, v.y, acc[RB - 1]);
                            }
                        }
                    }
                } else {  // Bernoulli (RB = 1, 2) or ACWB (RB = 2)
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        const int i = i0 + e * T;
                        if (i < n && BERN) {
                            // f += nu b_k* (line 10), r = y - sigma(f) (line 4 of the next iteration), log-loss
#pragma unroll
                            for (int q = 0; q < RB; q++) {
                                const double f = Fb[i * RB + q] + zhat[q * nsp + (q ? j1[e] : j0[e])];
                                Fb[i * RB + q] = f;
                                const double y = Yb[i * RB + q];
                                double lo;
                                const double v = bern_resid(y, f, &lo);
                                r[i * RB + q] = v;
                                acc[q] = fma(v, v, acc[q]);
                                accL[q] += lo;
                            }
                        } else if (i < n && ACC) {
                            const double2 v = *reinterpret_cast<double2*>(r + 2 * i);
                            const double bc = zhat[nsp + j1[e]];
                            const double F = v.x - zhat[j0[e]];
                            const double H = Hm[i] - eta * bc;
                            const double rn = (1.0 - vt1) * F + vt1 * H;
                            const double cn = rn + a1 * (v.y - bc);
                            Hm[i] = H;
                            *reinterpret_cast<double2*>(r + 2 * i) = make_double2(rn, cn);
                            accF = fma(F, F, accF);
                            acc[0] = fma(rn, rn, acc[0]);
                            acc[RB - 1] = fma(cn, cn, acc[RB - 1]);
                        }
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < RB; q++) red[(parw * NRB + q) * T + tid] = acc[q];
            if (ACC) red[(parw * NRB + RB) * T + tid] = accF;
            if (BERN)
#pragma unroll
                for (int q = 0; q < RB; q++) red[(parw * NRB + RB + q) * T + tid] = accL[q];
        }
        __syncthreads();
        if (timed) tm = phase_mark(&tD, tm, true);
        CWB_JIT(m * 8 + 6);
    }
    if (HC) {
        if (p.M > 0 && warp == 0) bookkeeping_hc(p.M - 1);
    } else if (ACC) {
        if (p.M > 0 && warp == 0) bookkeeping_acc(p.M - 1);
    } else if (p.M > 0 && warp < RB) {
        bookkeeping(p.M - 1, warp);
    }
    __syncthreads();  // agg complete
    if (ACC) {
        if (b0 < p.B) {
            for (int a = tid; a < K * d; a += T) {
                p.agg_out[(size_t)b0 * K * d + a] = agg[a];
                if (p.agg2_out) p.agg2_out[(size_t)b0 * K * d + a] = agg[K * d + a];
            }
            if (tid == 0 && p.offset_out) p.offset_out[b0] = f0[0];
            if (HC && tid == 0 && p.switch_iter) p.switch_iter[b0] = hc_sw;
        }
    } else {
#pragma unroll
        for (int q = 0; q < RB; q++)
            if (b0 + q < p.B) {
                for (int a = tid; a < K * d; a += T) p.agg_out[(size_t)(b0 + q) * K * d + a] = agg[q * K * d + a];
                if (tid == 0 && p.offset_out) p.offset_out[b0 + q] = f0[q];
            }
    }
    if (timed) {
        p.timing[0] = tA; p.timing[1] = tB; p.timing[2] = tC; p.timing[3] = tD;
    }
}

// ------------------------------------------------------------- plan kernel
// In-place exclusive scan of a[0..N) by the whole block; returns the total.
__device__ int block_scan_excl(int* a, int N, int* wsum) {
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, w = tid >> 5;
    const int per = (N + nthr - 1) / nthr;
    const int g0 = min(N, tid * per), g1 = min(N, g0 + per);
    int local = 0;
    for (int g = g0; g < g1; g++) local += a[g];
    int inc = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    __syncthreads();
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    if (w == 0) {
        int v = lane < (nthr >> 5) ? wsum[lane] : 0;
        int s = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += t;
        }
        wsum[lane] = s - v;
        if (lane == 31) wsum[32] = s;
    }
    __syncthreads();
    int run = wsum[w] + inc - local;
    for (int g = g0; g < g1; g++) {
        const int v = a[g];
        a[g] = run;
        run += v;
    }
    const int total = wsum[32];
    __syncthreads();
    return total;
}

// Plan, step 1 (one block).  Cuts every non-empty bin into ceil(count / P)
// tasks, sorts the tasks by length (descending, ties by bin order; coarse
// buckets), deals them to the T threads of the fused kernel in snake order and
// groups the rows of every task by colour (bank group, row mod G) for the
// scheduler.  Deterministic; runs once per (data set, RB, T).
template <typename SrcPermT>
__global__ void k_fused_plan(const int32_t* __restrict__ off, const SrcPermT* __restrict__ perm, int K, int ns,
                             int nsp, int n, int T, int P, int G, int32_t* __restrict__ plan,
                             int32_t* __restrict__ scratch, const int* status) {
    extern __shared__ int psm[];
    __shared__ int wsum[33];
    __shared__ unsigned hist[1024], run_b[1024];
    if (status && *status) return;
    const int KS = K * ns, NW = T / 32;
    const int tid = threadIdx.x, nthr = blockDim.x;
    int* pcs = psm;            // pieces per bin
    int* first = psm + KS;     // first task index of the bin
    int* slot = psm + 2 * KS;  // first piece slot (split bins)
    int* cidx = psm + 3 * KS;  // combine index (split bins)
    const int RM = plan_rounds_max(KS, T);
    int32_t* tt_dest = plan + 8;
    int32_t* wl = tt_dest + RM * T;
    int32_t* wb = wl + RM * NW;
    int32_t* comb_g = wb + RM * NW;
    int32_t* comb_first = comb_g + KS;
    int32_t* comb_cnt = comb_first + KS;
    const int n_tasks_max = KS + 2 * T;
    int32_t* s_start = scratch;
    int32_t* s_len = s_start + n_tasks_max;
    int32_t* s_dest = s_len + n_tasks_max;
    int32_t* s_bkt = s_dest + n_tasks_max;
    int32_t* s_slot = s_bkt + n_tasks_max;  // rd * T + thread of each task
    int32_t* s_tos = s_slot + n_tasks_max;  // task of each (rd, thread) slot, -1: none
    int32_t* cs = s_tos + RM * T;           // per task: 17 colour offsets
    int32_t* srt = cs + 17 * (size_t)n_tasks_max;  // task rows sorted by colour (K*n)
    for (int g = tid; g < KS; g += nthr) {
        const int k = g / ns, l = g - k * ns;
        const int c = off[k * (ns + 1) + l + 1] - off[k * (ns + 1) + l];
        const int pc = c > 0 ? (c + P - 1) / P : 0;
        pcs[g] = pc;
        first[g] = pc;
        slot[g] = pc > 1 ? pc : 0;
        cidx[g] = pc > 1 ? 1 : 0;
    }
    for (int e = tid; e < RM * T; e += nthr) { tt_dest[e] = kDiscard; s_tos[e] = -1; }
    for (int e = tid; e < 2 * RM * NW; e += nthr) wl[e] = 0;
    for (int e = tid; e < 1024; e += nthr) { hist[e] = 0; run_b[e] = 0; }
    __syncthreads();
    const int n_tasks = block_scan_excl(first, KS, wsum);
    const int n_multi = block_scan_excl(slot, KS, wsum);
    const int n_comb = block_scan_excl(cidx, KS, wsum);
    for (int g = tid; g < KS; g += nthr) {
        const int k = g / ns, l = g - k * ns;
        const int pc = pcs[g];
        if (pc == 0) continue;
        const int a0 = off[k * (ns + 1) + l], c = off[k * (ns + 1) + l + 1] - a0;
        const int ug = k * nsp + l;  // u index (rows of U padded to nsp)
        if (pc > 1) {
            comb_g[cidx[g]] = ug;
            comb_first[cidx[g]] = slot[g];
            comb_cnt[cidx[g]] = pc;
        }
        const int base = c / pc, rem = c % pc;
        int st = k * n + a0;
        for (int q = 0; q < pc; q++) {
            const int len = base + (q < rem ? 1 : 0);
            const int t = first[g] + q;
            s_start[t] = st;
            s_len[t] = len;
            s_dest[t] = pc == 1 ? ug : -(slot[g] + q) - 1;
            const int bk = (int)(((long long)len * 1024) / (P + 1));
            s_bkt[t] = 1023 - min(1023, bk);  // ascending key = descending length
            st += len;
        }
    }
    __syncthreads();
    for (int t = tid; t < n_tasks; t += nthr) {  // rows of every task grouped by colour (stable)
        const int st = s_start[t], len = s_len[t];
        int cnt[17];
        for (int c = 0; c <= G; c++) cnt[c] = 0;
        for (int q = 0; q < len; q++) cnt[(int)perm[st + q] % G + 1]++;
        for (int c = 0; c < G; c++) cnt[c + 1] += cnt[c];
        for (int c = 0; c <= G; c++) cs[t * 17 + c] = cnt[c];
        for (int q = 0; q < len; q++) {
            const int row = (int)perm[st + q];
            srt[st + cnt[row % G]++] = row;
        }
    }
    for (int t = tid; t < n_tasks; t += nthr) atomicAdd(&hist[s_bkt[t]], 1u);
    __syncthreads();
    if (tid < 32) {  // exclusive scan of the 1024 bucket counts (one warp, 32 per lane)
        unsigned loc = 0;
        for (int q = 0; q < 32; q++) loc += hist[tid * 32 + q];
        unsigned inc = loc;
        for (int o = 1; o < 32; o <<= 1) {
            unsigned v = __shfl_up_sync(0xffffffffu, inc, o);
            if (tid >= o) inc += v;
        }
        unsigned runv = inc - loc;
        for (int q = 0; q < 32; q++) {
            const unsigned h = hist[tid * 32 + q];
            hist[tid * 32 + q] = runv;
            runv += h;
        }
    }
    __syncthreads();
    if (tid < 32) {  // stable ranks within a bucket (task order), 32 tasks at a time
        for (int t0 = 0; t0 < n_tasks; t0 += 32) {
            const int t = t0 + tid;
            const bool valid = t < n_tasks;
            const unsigned bk = valid ? (unsigned)s_bkt[t] : 0xffffffffu;
            const unsigned mask = __match_any_sync(0xffffffffu, bk);
            const unsigned lt = mask & ((1u << tid) - 1u);
            if (valid) {
                const int srk = (int)(hist[bk] + run_b[bk] + __popc(lt));
                // snake order with the longest tasks on the HIGHEST thread ids (the warp
                // scheduler issues highest-warp-id first: critical-path warps get priority)
                const int rd = srk / T, i = srk - rd * T;
                const int th = (rd & 1) ? i : (T - 1 - i);
                tt_dest[rd * T + th] = s_dest[t];
                s_slot[t] = rd * T + th;
                s_tos[rd * T + th] = t;
            }
            __syncwarp();
            if (valid && lt == 0) run_b[bk] += __popc(mask);
            __syncwarp();
        }
    }
    __syncthreads();
    if (tid == 0) {
        plan[0] = n_tasks;
        plan[2] = n_comb;
        plan[3] = n_multi;
        plan[4] = P;
    }
}

// Plan, step 2: conflict-free gather schedule of one lane group (the G lanes that
// share a shared-memory wavefront: G = 16 for 8-byte rows, 8 for 16-byte rows).
// Colour of a row = its bank group (row mod G).  Every step each lane emits one
// row of its task or a zero padding row, and the G rows of a step have distinct
// colours, so each gather instruction is conflict-free.  The G lanes cooperate
// through segmented shuffles; each keeps its colour counts in registers.  Per
// step the lane with the most rows left picks first (so the longest task makes
// progress every step), then the others in rotated lane order; a lane takes the
// free colour it holds most rows of; lanes without a pick get the remaining free
// colours as padding rows.  The schedule goes to scratch ([group][step][G]).
template <int G>
__global__ void k_fused_sched(const int32_t* __restrict__ plan, const int32_t* __restrict__ scratch, int T, int KS,
                              int SB, int n_groups, int32_t* __restrict__ sched, int32_t* __restrict__ gsteps,
                              int* status) {
    if (status && *status) return;
    const int gt = blockIdx.x * blockDim.x + threadIdx.x;
    const int gi = gt / G, L = gt % G, lane = threadIdx.x & 31;
    const int RM = plan_rounds_max(KS, T);
    const int n_tasks_max = KS + 2 * T;
    const int32_t* s_start = scratch;
    const int32_t* s_tos = scratch + 5 * (size_t)n_tasks_max;
    const int32_t* cs = s_tos + RM * T;
    const bool valid = gi < n_groups;
    int t = -1;
    if (valid) {
        const int rd = gi / (T / G), th0 = (gi - rd * (T / G)) * G;
        t = s_tos[rd * T + th0 + L];
    }
    int rem[G], nxt[G], tot = 0;  // rows left per colour, next srt index per colour
#pragma unroll
    for (int c = 0; c < G; c++) {
        const int c0 = t >= 0 ? cs[t * 17 + c] : 0;
        const int c1 = t >= 0 ? cs[t * 17 + c + 1] : 0;
        rem[c] = c1 - c0;
        nxt[c] = (t >= 0 ? s_start[t] : 0) + c0;
        tot += rem[c];
    }
    const unsigned seg = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << (lane & ~(G - 1));
    int step = 0, gst = 0;
    for (;;) {
        const unsigned act = __ballot_sync(0xffffffffu, tot > 0);
        if (!act) break;  // warp-uniform loop: shuffles stay convergent
        const bool seg_active = (act & seg) != 0u;
        // first pick: most rows left, ties lowest lane
        int key = tot > 0 ? (tot << 5) | (31 - L) : -1;
        for (int o = 1; o < G; o <<= 1) key = max(key, __shfl_xor_sync(0xffffffffu, key, o, G));
        const int first = key >= 0 ? 31 - (key & 31) : 0;
        unsigned taken = 0u;
        int mycol = -1;
#pragma unroll 1
        for (int e = 0; e < G; e++) {
            const int cur = (first + e) % G;
            // most rows among the free colours, ties lowest colour: max of packed keys
            // (rem << 4 | 15 - c), reduced as a tree to keep the dependent chain short
            int kv[G];
#pragma unroll
            for (int c = 0; c < G; c++) kv[c] = ((taken >> c) & 1u) ? 0 : (rem[c] << 4) | (15 - c);
#pragma unroll
            for (int w = G / 2; w > 0; w >>= 1)
#pragma unroll
                for (int c = 0; c < w; c++) kv[c] = max(kv[c], kv[c + w]);
            int pick = (L == cur && tot > 0 && (kv[0] >> 4) > 0) ? 15 - (kv[0] & 15) : -1;
            pick = __shfl_sync(0xffffffffu, pick, cur, G);
            if (pick >= 0) {
                taken |= 1u << pick;
                if (L == cur) mycol = pick;
            }
        }
        int mypick = -1;  // -> srt index of the row
        if (mycol >= 0) {
#pragma unroll
            for (int c = 0; c < G; c++)
                if (c == mycol) { rem[c]--; mypick = nxt[c]++; }
            tot--;
        }
        // padding for lanes without a pick: the free colours in lane order (entry -1 - colour)
        const unsigned nop = __ballot_sync(0xffffffffu, mypick < 0) & seg;
        int entry = mypick;  // srt index of the row (resolved by k_fused_pack)
        if (mypick < 0) {
            int rank = __popc(nop & ((1u << lane) - 1u) & seg);
            unsigned freec = ~taken & ((1u << G) - 1u);
            for (; rank > 0; rank--) freec &= freec - 1u;
            entry = -__ffs(freec);  // -1 - colour
        }
        if (seg_active) {
            if (valid && step < SB) sched[((size_t)gi * SB + step) * G + L] = entry;
            if (valid && step >= SB && L == 0) cwb_dev_fail(status, CWB_ECUDA);  // bound exceeded
            gst = step + 1;
        }
        step += 1;
        if (step >= SB + 1) break;
    }
    if (valid && L == 0) gsteps[gi] = gst;  // steps of this group
}

// Plan, step 3 (one block): steps per warp and round (max over its lane groups,
// rounded up to 4), block offsets of the schedule, round count and size.
__global__ void k_fused_wl(int32_t* __restrict__ plan, const int32_t* __restrict__ gsteps, int KS, int T, int G,
                           const int* status) {
    if (status && *status) return;
    const int RM = plan_rounds_max(KS, T), NW = T / 32, gpw = 32 / G;
    int32_t* wl = plan + 8 + RM * T;
    int32_t* wb = wl + RM * NW;
    for (int e = threadIdx.x; e < RM * NW; e += blockDim.x) {
        int st = 0;
        for (int g = 0; g < gpw; g++) st = max(st, gsteps[e * gpw + g]);
        wl[e] = (st + 7) / 8 * 8;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int o = 0, rounds = 0;
        for (int e = 0; e < RM * NW; e++) {
            wb[e] = o;
            o += 32 * wl[e];
            if (wl[e]) rounds = e / NW + 1;
        }
        plan[1] = rounds;
        plan[5] = o;
    }
}

// Plan, step 4: the schedule in the kernel's layout ([step/4][lane][4] per warp
// and round block), padding steps beyond a group's schedule with zero rows of
// distinct colours.
template <typename PermT>
__global__ void k_fused_pack(const int32_t* __restrict__ plan, const int32_t* __restrict__ scratch,
                             const int32_t* __restrict__ sched, const int32_t* __restrict__ gsteps, int KS, int T,
                             int G, int SB, int n, int stride, PermT* __restrict__ permt, const int* status) {
    if (status && *status) return;
    const int RM = plan_rounds_max(KS, T), NW = T / 32;
    const int32_t* srt = scratch + 22 * (size_t)(KS + 2 * T) + (size_t)RM * T;  // task rows by colour
    const int32_t* wl = plan + 8 + RM * T;
    const int32_t* wb = wl + RM * NW;
    const int rounds = plan[1];
    for (int e = blockIdx.x; e < rounds * NW; e += gridDim.x) {
        const int steps = wl[e];
        for (int x = threadIdx.x; x < steps * 32; x += blockDim.x) {
            const int st = x >> 5, ln = x & 31;
            const int gi = e * (32 / G) + ln / G, L = ln % G;
            int v;
            const int x2 = st < gsteps[gi] ? sched[((size_t)gi * SB + st) * G + L] : -1 - L;
            const int row = x2 >= 0 ? srt[x2] : n + (((-1 - x2 - n) % G) + G) % G;
            v = stride * row;
            permt[(size_t)wb[e] + (size_t)(st >> 2) * 128 + ln * 4 + (st & 3)] = (PermT)v;
        }
    }
}

template <typename IdxT, typename PermT, int RB, bool POOL, int MAXT, int MINB, bool ACC = false, bool HC = false,
          bool BERN = false>
int launch_t(const FusedParams& fp, int T, size_t smem, cudaStream_t s) {
    auto kern = k_train_fused<IdxT, PermT, RB, POOL, MAXT, MINB, ACC, HC, BERN>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return -1;
    const int grid = ACC ? fp.B : (fp.B + RB - 1) / RB;
    kern<<<grid, T, smem, s>>>(fp);
    return 0;
}

template <typename IdxT, typename PermT>
int launch_sel(const FusedParams& fp, int T, int RB, bool pool, size_t smem, cudaStream_t s, bool acc = false,
               bool hc = false, bool bern = false) {
    if (bern) {  // Bernoulli loss: the CWB shapes of k_train_fused plus y and f in shared memory
        if (RB == 2) {
            if (pool) return launch_t<IdxT, PermT, 2, true, 512, 1, false, false, true>(fp, T, smem, s);
            return launch_t<IdxT, PermT, 2, false, 512, 1, false, false, true>(fp, T, smem, s);
        }
        if (pool) return launch_t<IdxT, PermT, 1, true, 768, 1, false, false, true>(fp, T, smem, s);
        return launch_t<IdxT, PermT, 1, false, 768, 1, false, false, true>(fp, T, smem, s);
    }
    if (hc) {  // HCWB: the ACWB layout plus F, the validation mask and the phase state
        if (T <= 256) {
            if (pool) return launch_t<IdxT, PermT, 2, true, 256, 2, true, true>(fp, T, smem, s);
            return launch_t<IdxT, PermT, 2, false, 256, 2, true, true>(fp, T, smem, s);
        }
        if (pool) return launch_t<IdxT, PermT, 2, true, 512, 1, true, true>(fp, T, smem, s);
        return launch_t<IdxT, PermT, 2, false, 512, 1, true, true>(fp, T, smem, s);
    }
    if (acc) {  // ACWB: two columns of one replication; 512 threads, or 256 with two CTAs per SM
        if (T <= 256) {
            if (pool) return launch_t<IdxT, PermT, 2, true, 256, 2, true>(fp, T, smem, s);
            return launch_t<IdxT, PermT, 2, false, 256, 2, true>(fp, T, smem, s);
        }
        if (pool) return launch_t<IdxT, PermT, 2, true, 512, 1, true>(fp, T, smem, s);
        return launch_t<IdxT, PermT, 2, false, 512, 1, true>(fp, T, smem, s);
    }
    if (RB == 2) {
        if (T == 384) {  // register-resident A^-1 columns (AREG_T)
            if (pool) return launch_t<IdxT, PermT, 2, true, 384, 1>(fp, T, smem, s);
            return launch_t<IdxT, PermT, 2, false, 384, 1>(fp, T, smem, s);
        }
        if (T > 512) {
            if (pool) return launch_t<IdxT, PermT, 2, true, 768, 1>(fp, T, smem, s);
            return launch_t<IdxT, PermT, 2, false, 768, 1>(fp, T, smem, s);
        }
        if (pool) return launch_t<IdxT, PermT, 2, true, 512, 1>(fp, T, smem, s);
        return launch_t<IdxT, PermT, 2, false, 512, 1>(fp, T, smem, s);
    }
    if (T <= 384) {
        if (pool) return launch_t<IdxT, PermT, 1, true, 384, 2>(fp, T, smem, s);
        return launch_t<IdxT, PermT, 1, false, 384, 2>(fp, T, smem, s);
    }
    if (pool) return launch_t<IdxT, PermT, 1, true, 768, 1>(fp, T, smem, s);
    return launch_t<IdxT, PermT, 1, false, 768, 1>(fp, T, smem, s);
}

}  // namespace

static const size_t kMaxSmem = 227 * 1024;
static const size_t kTwoCtaSmem = 113 * 1024;

struct FusedShape {
    int RB = 0, T = 0, P = 0, permt_bytes = 2;
    bool pool = false;
    size_t cap = 0, smem = 0;
};

// Launch shape for B replications: RB replications per CTA, T threads, pool
// tables in shared memory or not.  false when the residuals do not fit.
static bool fused_shape(const cwb_ctx* c, int B, FusedShape* out, bool bern = false) {
    if ((int64_t)c->K * c->n + 8 > INT32_MAX) return false;
    if ((int64_t)c->K * c->n_star * 16 > 200 * 1024) return false;  // plan kernel shared memory
    const int KS = c->K * c->n_star;
    struct Cand { int RB, T; size_t lim; };
    Cand cands[4];
    int nc = 0;
    const int nsm = cwb_num_sms();
    // 384 threads (the register-resident A^-1 instance) when every learner gets its own warp at d = 24, else 512
    static const int t2env = getenv("CWB_FT2") ? atoi(getenv("CWB_FT2")) : 0;  // experiments only
    const int t2 = t2env ? t2env : ((!bern && c->K <= 12 && c->d == kAregD) ? 384 : 512);
    static const int t1 = getenv("CWB_FT1") ? atoi(getenv("CWB_FT1")) : 0;
    if (B > nsm) cands[nc++] = {2, t2, kMaxSmem};  // ~2 replications per SM: one CTA (512 best of 256..768)
    if (B > nsm && !bern) cands[nc++] = {1, std::min(384, std::max(256, 32 * c->K)), kTwoCtaSmem};
    cands[nc++] = {1, t1 ? t1 : (c->n >= 8192 ? 768 : 512), kMaxSmem};
    for (int i = 0; i < nc; i++) {
        FusedShape f;
        f.RB = cands[i].RB;
        f.T = cands[i].T;
        const int64_t stride = 8 * f.RB;
        f.permt_bytes = stride * (c->n + kPadRows) <= 65535 ? 2 : 4;
        // task size: balance the K*n rows over T threads, but do not cut bins of up to
        // piece_factor() x the mean bin size (a cut bin costs a combine pass)
        f.P = std::max(4, (int)std::max((c->K * c->n + f.T - 1) / f.T, (int64_t)(piece_factor() * c->n / c->n_star)));
        f.cap = permt_bound(KS, f.T, f.P);
        for (int pool = 1; pool >= 0; pool--) {
            SmemLayout L((int)c->n, c->K, c->nsp, c->d, c->W, 2 * f.T, f.RB, f.T / 32, pool != 0, f.cap * f.permt_bytes, 0,
                         1, false, false, bern);
            if (L.total <= cands[i].lim) {
                f.pool = pool != 0;
                f.smem = L.total;
                *out = f;
                return true;
            }
        }
    }
    return false;
}

size_t cwb_fused_smem_bytes(const cwb_ctx* c) {
    FusedShape f;
    return fused_shape(c, 1, &f) ? f.smem : (size_t)-1;
}

// (Re)builds the H1 task plan for the shape of a B-replication launch.
// Pinned host slots for the plan headers (read back without a synchronous copy).  A slot belongs
// to one context from its first plan until cwb_free (cwb_release_header_slot); slots come from
// pinned chunks of 256, allocated on demand, so live contexts never share one.
namespace {
std::mutex g_hdr_mu;
std::vector<int32_t*> g_hdr_free;
}  // namespace

static int32_t* pinned_header_slot() {
    std::lock_guard<std::mutex> lock(g_hdr_mu);
    if (g_hdr_free.empty()) {
        void* p = nullptr;
        if (cudaHostAlloc(&p, sizeof(int32_t) * 16 * 256, cudaHostAllocDefault) != cudaSuccess) return nullptr;
        for (int i = 255; i >= 0; i--) g_hdr_free.push_back((int32_t*)p + 16 * i);
    }
    int32_t* slot = g_hdr_free.back();
    g_hdr_free.pop_back();
    return slot;
}

void cwb_release_header_slot(int32_t* slot) {
    if (!slot) return;
    std::lock_guard<std::mutex> lock(g_hdr_mu);
    g_hdr_free.push_back(slot);
}

// Launches the H1 plan for launch shape f on stream s (allocations stream-ordered on s):
// k_fused_plan -> k_fused_sched -> k_fused_wl -> k_fused_pack into a schedule buffer of bound
// size, then an asynchronous copy of the header and the device status to a pinned slot and
// an event.  No host synchronisation: fused_plan_finish reads the header when it is needed.
static int fused_plan_launch(cwb_ctx* c, const FusedShape& f, cudaStream_t s) {
    if (c->ev_plan) CWB_CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_plan, 0));  // previous plan may still build
    cwb_release(c->plan, s);
    cwb_release(c->permt, s);
    c->plan = nullptr;
    c->permt = nullptr;
    c->fused_T = 0;
    c->plan_pending = false;
    const int KS = c->K * c->n_star, T = f.T, G = 16 / f.RB;
    const int RM = plan_rounds_max(KS, T), NW = T / 32;
    const int n_groups = RM * T / G;
    const int SB = 2 * ((f.P + 3) / 4 * 4) + G;  // schedule steps bound per group
    const size_t scratch_ints = 22 * (size_t)(KS + 2 * T) + (size_t)RM * T + (size_t)c->K * c->n;
    const size_t sched_ints = (size_t)n_groups * SB * G + n_groups;
    const size_t permt_cap = (size_t)RM * T * ((SB + 7) / 8 * 8) + kSlackEntries;
    if (!c->h_hdr) c->h_hdr = pinned_header_slot();
    if (!c->h_hdr) return cwb_set_error(c, CWB_ENOMEM, "pinned header allocation failed");
    if (!c->ev_plan && cudaEventCreateWithFlags(&c->ev_plan, cudaEventDisableTiming) != cudaSuccess)
        return cwb_set_error(c, CWB_ECUDA, "event creation failed");
    if (cwb_alloc((void**)&c->plan, sizeof(int32_t) * (plan_ints(KS, T) + scratch_ints + sched_ints), s) != cudaSuccess ||
        cwb_alloc(&c->permt, (size_t)f.permt_bytes * permt_cap, s) != cudaSuccess)
        return cwb_set_error(c, CWB_ENOMEM, "fused plan allocation failed");
    int32_t* scratch = c->plan + plan_ints(KS, T);
    int32_t* sched = scratch + scratch_ints;
    int32_t* gsteps = sched + (size_t)n_groups * SB * G;
    const size_t psmem = sizeof(int) * 4 * (size_t)KS;
    const int stride = 8 * f.RB;
    if (c->perm_bytes == 2) {
        auto kern = k_fused_plan<uint16_t>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem);
        kern<<<1, 1024, psmem, s>>>(c->off, (const uint16_t*)c->perm, c->K, c->n_star, c->nsp, (int)c->n, T, f.P, G,
                                    c->plan, scratch, c->d_status);
    } else {
        auto kern = k_fused_plan<uint32_t>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem);
        kern<<<1, 1024, psmem, s>>>(c->off, (const uint32_t*)c->perm, c->K, c->n_star, c->nsp, (int)c->n, T, f.P, G,
                                    c->plan, scratch, c->d_status);
    }
    const int sthreads = n_groups * G;  // one warp per block: spread the latency-bound groups over the SMs
    if (G == 8)
        k_fused_sched<8><<<(sthreads + 31) / 32, 32, 0, s>>>(c->plan, scratch, T, KS, SB, n_groups, sched, gsteps,
                                                             c->d_status);
    else
        k_fused_sched<16><<<(sthreads + 31) / 32, 32, 0, s>>>(c->plan, scratch, T, KS, SB, n_groups, sched, gsteps,
                                                              c->d_status);
    k_fused_wl<<<1, 256, 0, s>>>(c->plan, gsteps, KS, T, G, c->d_status);
    const int blocks = std::max(1, std::min(RM * NW, 1184));
    if (f.permt_bytes == 2)
        k_fused_pack<uint16_t><<<blocks, 256, 0, s>>>(c->plan, scratch, sched, gsteps, KS, T, G, SB, (int)c->n,
                                                      stride, (uint16_t*)c->permt, c->d_status);
    else
        k_fused_pack<uint32_t><<<blocks, 256, 0, s>>>(c->plan, scratch, sched, gsteps, KS, T, G, SB, (int)c->n,
                                                      stride, (uint32_t*)c->permt, c->d_status);
    c->launches += 4;
    CWB_CUDA_TRY(c, cudaMemcpyAsync(c->h_hdr, c->plan, sizeof(int32_t) * 8, cudaMemcpyDeviceToHost, s));
    CWB_CUDA_TRY(c, cudaMemcpyAsync(c->h_hdr + 8, c->d_status, sizeof(int), cudaMemcpyDeviceToHost, s));
    CWB_CUDA_TRY(c, cudaEventRecord(c->ev_plan, s));
    int rc = cwb_check_launch(c, "fused plan kernels");
    if (rc) return rc;
    c->plan_pending = true;
    c->plan_T = T;
    c->plan_rb = f.RB;
    c->plan_permt_bytes = f.permt_bytes;
    c->plan_cap = permt_cap;
    return CWB_OK;
}

// Waits for the plan (host), takes over its header.
static int fused_plan_finish(cwb_ctx* c) {
    if (!c->plan_pending) return CWB_OK;
    CWB_CUDA_TRY(c, cudaEventSynchronize(c->ev_plan));
    c->plan_pending = false;
    const int32_t* hdr = c->h_hdr;
    if (hdr[8]) return CWB_OK;  // device error: reported by cwb_status
    if ((size_t)hdr[5] + kSlackEntries > c->plan_cap) return cwb_set_error(c, CWB_ECUDA, "fused plan exceeds its bound");
    c->fused_T = c->plan_T;
    c->fused_rb = c->plan_rb;
    c->permt_bytes = c->plan_permt_bytes;
    c->permt_entries = hdr[5];
    c->plan_multi = hdr[3];
    return CWB_OK;
}

// Shape (replications and threads per CTA, task size) of a fused launch of B replications for the
// CWB (acc = false), ACWB / HCWB (acc, hc) or Bernoulli (bern) kernel; false when it does not fit.
static bool train_shape(const cwb_ctx* c, int B, bool acc, bool hc, bool bern, FusedShape* out) {
    if (!acc) return fused_shape(c, B, out, bern);
    FusedShape f;  // the two columns (r, c) of a replication run as RB = 2
    if ((int64_t)c->K * c->n + 8 > INT32_MAX || (int64_t)c->K * c->n_star * 16 > 200 * 1024) return false;
    f.RB = 2;
    f.permt_bytes = 16 * (c->n + kPadRows) <= 65535 ? 2 : 4;
    // HCWB with more replications than SMs: 256-thread CTAs, two per SM, when both fit in shared
    // memory (R1: 3.24 -> 2.98 ms; ACWB measured slower that way, 2.33 -> 2.48 ms, and keeps
    // 512).  CWB_ACC_T=256|512 overrides.
    const char* ev = getenv("CWB_ACC_T");
    const int want = ev ? atoi(ev) : (hc && B > cwb_num_sms() ? 256 : 512);
    f.T = 0;
    for (int T : {256, 512}) {
        if (T < want) continue;
        const size_t lim = T == 256 ? kTwoCtaSmem : kMaxSmem;
        if (SmemLayout((int)c->n, c->K, c->nsp, c->d, c->W, 2 * T, 2, T / 32, false, 0, 0, c->idx_bytes, true,
                       hc)
                .total <= lim) {
            f.T = T;
            break;
        }
    }
    if (!f.T) return false;
    f.P = std::max(4, (int)std::max((c->K * c->n + f.T - 1) / f.T, (int64_t)(piece_factor() * c->n / c->n_star)));
    *out = f;
    return true;
}

// Pre-builds the plan for the expected batch (cwb_config.batch_hint) on a side stream that
// starts right after the bin inversion, so it overlaps the basis / binMatMat / df->lambda
// kernels of cwb_init.  Called by cwb_launch_init after k_csr.
int cwb_fused_plan(cwb_ctx* c, cudaStream_t s) {
    if (c->batch_hint <= 0) return CWB_OK;
    FusedShape f;  // the shape of the training call the hint names (cwb_config.train_hint)
    const int th = c->train_hint;
    if (!train_shape(c, c->batch_hint, th == 1 || th == 2, th == 2, th == 3, &f)) return CWB_OK;
    if (!c->s2) {  // one side stream per device, shared by the contexts (created once, never destroyed)
        static cudaStream_t side[16] = {};
        static std::mutex mu;
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return CWB_OK;
        std::lock_guard<std::mutex> lock(mu);
        if (!side[dev] && cudaStreamCreateWithFlags(&side[dev], cudaStreamNonBlocking) != cudaSuccess) return CWB_OK;
        c->s2 = side[dev];
    }
    if (!c->ev_csr && cudaEventCreateWithFlags(&c->ev_csr, cudaEventDisableTiming) != cudaSuccess) return CWB_OK;
    CWB_CUDA_TRY(c, cudaEventRecord(c->ev_csr, s));
    CWB_CUDA_TRY(c, cudaStreamWaitEvent(c->s2, c->ev_csr, 0));
    return fused_plan_launch(c, f, c->s2);
}

// Shared host path of the fused CWB (acc = false) and ACWB (acc = true) launches.
struct HcArgs {  // HCWB extras of a fused launch
    const uint8_t* vmask = nullptr;
    const double* Ainv_tr = nullptr;
    const double* Cb_tr = nullptr;
    int pat0 = 0;
    double* val_risk_trace = nullptr;
    int32_t* switch_iter = nullptr;
};

static int train_fused_common(cwb_ctx* c, bool acc, const double* Y, int32_t B, double nu, double gamma, int32_t M,
                              double* offset_out, double* theta_out, double* theta_h_out, int32_t* k_trace,
                              int32_t* kcor_trace, double* sse_trace, double* risk_trace, cudaStream_t s,
                              bool* launched, const HcArgs* hc = nullptr, bool bern = false) {
    *launched = false;
    FusedShape f;
    if (!train_shape(c, B, acc, hc != nullptr, bern, &f)) return CWB_OK;  // does not fit: general path
    int rc = CWB_OK;
    const bool have = (c->plan_pending && c->plan_T == f.T && c->plan_rb == f.RB) ||
                      (!c->plan_pending && c->fused_T == f.T && c->fused_rb == f.RB && c->plan);
    if (!have) rc = fused_plan_launch(c, f, s);
    if (rc) return rc;
    rc = fused_plan_finish(c);
    if (rc) return rc;
    if (c->fused_T != f.T) return CWB_OK;  // plan failed on the device: cwb_status reports it
    CWB_CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_plan, 0));  // the plan may come from the side stream
    const size_t lim = ((f.RB == 1 || acc) && f.T <= 384) ? kTwoCtaSmem : kMaxSmem;
    const size_t pbytes = ((size_t)(c->permt_entries + kSlackEntries) * f.permt_bytes + 15) / 16 * 16;  // < plan_cap
    f.pool = false;
    const int nm = c->plan_multi;
    const bool hcm = hc != nullptr;
    f.smem = SmemLayout((int)c->n, c->K, c->nsp, c->d, c->W, nm, f.RB, f.T / 32, false, 0, 0, c->idx_bytes, acc,
                        hcm, bern).total;
    if (f.smem > lim) return CWB_OK;
    int ztab = 0;
    {   // POOL: schedule, B tables, Zs / zj0 and the index vectors all in shared memory, or none
        SmemLayout L1((int)c->n, c->K, c->nsp, c->d, c->W, nm, f.RB, f.T / 32, true, pbytes, 3, c->idx_bytes, acc,
                      hcm, bern);
        if (L1.total <= lim) {
            f.pool = true;
            ztab = 3;
            f.smem = L1.total;
        }
    }
    FusedParams fp;
    fp.n = (int)c->n; fp.K = c->K; fp.ns = c->n_star; fp.nsp = c->nsp; fp.d = c->d; fp.M = M; fp.B = B; fp.nu = nu;
    fp.gamma = gamma;
    fp.n_multi = c->plan_multi;
    fp.ztab = ztab;
    fp.permt_cap = (int)(pbytes / f.permt_bytes);
    fp.Y = Y; fp.idx = c->idx; fp.permt = c->permt; fp.plan = c->plan; fp.zj0 = c->zj0; fp.Zs = c->Zs;
    fp.inv2n = 1.0 / (2.0 * (double)c->n);
    fp.ZT = c->ZT; fp.lwin = c->lwin; fp.Ainv = c->Ainv; fp.Cb = c->Cb; fp.W = c->W;
    fp.offset_out = offset_out; fp.agg_out = theta_out; fp.agg2_out = theta_h_out;
    fp.k_trace = k_trace; fp.kcor_trace = kcor_trace; fp.sse_trace = sse_trace; fp.risk_trace = risk_trace;
    fp.timing = c->timing;
    fp.status = c->d_status;
    fp.vmask = nullptr; fp.Ainv_tr = nullptr; fp.Cb_tr = nullptr; fp.pat0 = 0;
    fp.val_risk_trace = nullptr; fp.switch_iter = nullptr;
    if (hcm) {
        fp.vmask = hc->vmask; fp.Ainv_tr = hc->Ainv_tr; fp.Cb_tr = hc->Cb_tr; fp.pat0 = hc->pat0;
        fp.val_risk_trace = hc->val_risk_trace; fp.switch_iter = hc->switch_iter;
    }
    const bool i8 = c->idx_bytes == 1, p16 = f.permt_bytes == 2;
    if (i8 && p16) rc = launch_sel<uint8_t, uint16_t>(fp, f.T, f.RB, f.pool, f.smem, s, acc, hcm, bern);
    else if (i8) rc = launch_sel<uint8_t, uint32_t>(fp, f.T, f.RB, f.pool, f.smem, s, acc, hcm, bern);
    else if (p16) rc = launch_sel<uint16_t, uint16_t>(fp, f.T, f.RB, f.pool, f.smem, s, acc, hcm, bern);
    else rc = launch_sel<uint16_t, uint32_t>(fp, f.T, f.RB, f.pool, f.smem, s, acc, hcm, bern);
    if (rc) return cwb_set_error(c, CWB_ECUDA, "fused kernel: cannot set shared memory size");
    c->launches++;
    c->fused_smem = f.smem;
    c->fused_pool = f.pool;
    *launched = true;
    return cwb_check_launch(c, "k_train_fused");
}

int cwb_train_fused(cwb_ctx* c, const double* Y, int32_t B, double nu, int32_t M, double* offset_out,
                    double* theta_agg_out, int32_t* k_trace, double* sse_trace, double* risk_trace,
                    cudaStream_t s, bool* launched) {
    return train_fused_common(c, false, Y, B, nu, 0.0, M, offset_out, theta_agg_out, nullptr, k_trace, nullptr,
                              sse_trace, risk_trace, s, launched);
}

int cwb_train_acwb_fused(cwb_ctx* c, const double* Y, int32_t B, double nu, double gamma, int32_t M,
                         double* offset_out, double* theta_f_out, double* theta_h_out, int32_t* k_trace,
                         int32_t* kcor_trace, double* sse_trace, double* risk_trace, cudaStream_t s,
                         bool* launched) {
    return train_fused_common(c, true, Y, B, nu, gamma, M, offset_out, theta_f_out, theta_h_out, k_trace,
                              kcor_trace, sse_trace, risk_trace, s, launched);
}

int cwb_train_hcwb_fused(cwb_ctx* c, const double* Y, int32_t B, const uint8_t* val_mask, const double* Ainv_tr,
                         const double* Cb_tr, double nu, double gamma, int32_t pat0, int32_t M, double* offset_out,
                         double* theta_f_out, int32_t* k_trace, int32_t* kcor_trace, double* sse_trace,
                         double* risk_trace, double* val_risk_trace, int32_t* switch_iter, cudaStream_t s,
                         bool* launched) {
    HcArgs h;
    h.vmask = val_mask; h.Ainv_tr = Ainv_tr; h.Cb_tr = Cb_tr; h.pat0 = pat0;
    h.val_risk_trace = val_risk_trace; h.switch_iter = switch_iter;
    return train_fused_common(c, true, Y, B, nu, gamma, M, offset_out, theta_f_out, nullptr, k_trace, kcor_trace,
                              sse_trace, risk_trace, s, launched, &h);
}

int cwb_train_bernoulli_fused(cwb_ctx* c, const double* Y, int32_t B, double nu, int32_t M, double* offset_out,
                              double* theta_agg_out, int32_t* k_trace, double* sse_trace, double* risk_trace,
                              cudaStream_t s, bool* launched) {
    return train_fused_common(c, false, Y, B, nu, 0.0, M, offset_out, theta_agg_out, nullptr, k_trace, nullptr,
                              sse_trace, risk_trace, s, launched, nullptr, true);
}
