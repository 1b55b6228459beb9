// cwb_fused.cu -- the whole CWB loop (Alg. 1 supp.) for one
// replication per CTA, all M iterations in one launch.
//
// Replications are independent boosting runs that share the binned pool, so
// a CTA never waits for another CTA: no grid barrier, no atomics, no host
// round trip between iterations.  The residual vector r (n doubles) and the
// bin sums u (K x n* doubles) stay in shared memory for all M iterations;
// the pool (task table, basis, cached inverse) is read-only and L1/L2
// resident.  Per iteration m:
//
//   H1  u_k(l) = sum_{i in bin l of learner k} r_i      binMatVec loop
//       The K*n* bins are cut into tasks of at most P rows (P ~ K n / T),
//       sorted by length and dealt to the T threads in snake order by a plan
//       built once per data set (k_fused_plan).  The row ids of the 32 tasks
//       of a warp are stored step-major ([step][lane], padded with a zero
//       row), so each step is one coalesced index load and one gather, with
//       no per-row branch; rows inside a task are ordered by shared-memory
//       bank (rotated per lane) so that the gathers of a step spread over the
//       banks.  A bin cut into several tasks is completed by a fixed-order
//       combine.
//   H2  s_k = Zb_k^T u_k  (4 non-zeros per design point)
//   H3  theta_k = (G_k + lambda_k D)^-1 s_k (cached)
//   H4  delta_k = 2 theta_k^T s_k - theta_k^T G_k theta_k,  SSE_k = r^T r - delta_k
//   H5  k* = argmin SSE_k = argmax delta_k, lowest k on ties
//   H6  r -= nu Zb_{k*}(idx_{k*}(i)) theta*;  theta_agg[k*] += nu theta*;  r^T r
//
// One warp per learner runs H2-H4 (lane j = coefficient j), so the solve and
// the SSE reduction use register shuffles instead of shared-memory passes.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "cwb_internal.cuh"

namespace {

constexpr int kDiscard = INT32_MIN;

struct FusedParams {
    int n, K, ns, d, M, B, T, n_multi;
    double nu;
    const double* Y;
    const void* idx;
    const void* permt;
    const int32_t* plan;
    const int32_t* zj0;
    const double* Zs;
    const double* Zb;
    const int32_t* lwin;
    const double* Ainv;
    const double* G;
    double* offset_out;
    double* agg_out;
    int32_t* k_trace;
    double* sse_trace;
    double* risk_trace;
    int* status;
};

__host__ __device__ __forceinline__ size_t align16(size_t b) { return (b + 15) & ~(size_t)15; }

struct SmemLayout {
    size_t r, U, th, delta, zhat, agg, pc, red, total;
    __host__ __device__ SmemLayout(int n, int K, int ns, int d, int T, int n_multi) {
        const size_t KS = (size_t)K * ns;
        size_t o = 0;
        r = o; o = align16(o + sizeof(double) * (n + 1));  // r[n] = 0: padding row
        U = o; o = align16(o + sizeof(double) * KS);
        th = o; o = align16(o + sizeof(double) * (size_t)K * 32);
        delta = o; o = align16(o + sizeof(double) * K);
        zhat = o; o = align16(o + sizeof(double) * ns);
        agg = o; o = align16(o + sizeof(double) * (size_t)K * d);
        pc = o; o = align16(o + sizeof(double) * (n_multi > 0 ? n_multi : 1));
        red = o; o = align16(o + sizeof(double) * 32);
        total = o;
    }
};

// plan layout (int32), built by k_fused_plan:
//   [0] n_tasks [1] rounds [2] n_comb [3] n_multi [4] P [5] permt entries [6..7] 0
//   tt_dest[R*T]   destination of thread t's task in round r (>= 0: u index,
//                  < 0: piece slot -dest-1, INT32_MIN: no task)
//   wl[R*NW]       steps of warp w in round r (multiple of 4, 0: none)
//   wb[R*NW]       offset of that block in permt ([step][lane] row ids)
//   comb_g[KS] comb_first[KS] comb_cnt[KS]   bins cut into several pieces
__host__ __device__ __forceinline__ int plan_rounds_max(int KS, int T) { return (KS + 2 * T) / T + 1; }
__host__ __device__ __forceinline__ size_t plan_ints(int KS, int T) {
    const size_t R = plan_rounds_max(KS, T);
    return 8 + R * T + 2 * R * (T / 32) + 3 * (size_t)KS;
}
__host__ __device__ __forceinline__ size_t permt_bound(int KS, int T, int P) {
    return (size_t)plan_rounds_max(KS, T) * T * (size_t)((P + 3) / 4 * 4);
}

template <typename IdxT, typename PermT, int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB) k_train_fused(FusedParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int T = blockDim.x, NW = T >> 5;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b = blockIdx.x;
    const int n = p.n;
    const int K = p.K, ns = p.ns, d = p.d, KS = K * ns;
    const SmemLayout L(n, K, ns, d, T, p.n_multi);
    double* r = (double*)(smem + L.r);
    double* U = (double*)(smem + L.U);
    double* th = (double*)(smem + L.th);
    double* delta = (double*)(smem + L.delta);
    double* zhat = (double*)(smem + L.zhat);
    double* agg = (double*)(smem + L.agg);
    double* pc = (double*)(smem + L.pc);
    double* red = (double*)(smem + L.red);
    const PermT* permt = (const PermT*)p.permt;
    const IdxT* idx = (const IdxT*)p.idx;

    // ---- prologue: plan tables, I8 offset f0 = mean(y) ---------------
    const int32_t* pl = p.plan;
    const int rounds = pl[1], n_comb = pl[2];
    const int RM = plan_rounds_max(KS, T);
    const int32_t* tt_dest = pl + 8;
    const int32_t* wl = tt_dest + RM * T;
    const int32_t* wb = wl + RM * NW;
    const int32_t* comb_g = wb + RM * NW;
    const int32_t* comb_first = comb_g + KS;
    const int32_t* comb_cnt = comb_first + KS;
    for (int a = tid; a < KS; a += T) U[a] = 0.0;  // empty bins keep u = 0
    for (int a = tid; a < K * d; a += T) agg[a] = 0.0;
    if (tid == 0) r[n] = 0.0;

    const double* y = p.Y + (size_t)b * n;
    double part = 0.0;
    bool bad = false;
    for (int i = tid; i < n; i += T) {
        double v = y[i];
        bad |= !isfinite(v);
        r[i] = v;
        part += v;
    }
    if (bad) cwb_dev_fail(p.status, CWB_ENONFINITE);
    part = warp_sum(part);
    if (lane == 0) red[warp] = part;
    __syncthreads();
    double sy = 0.0;
    for (int w = 0; w < NW; w++) sy += red[w];
    const double f0 = sy / (double)n;
    part = 0.0;
    for (int i = tid; i < n; i += T) {
        double v = r[i] - f0;
        r[i] = v;
        part += v * v;
    }
    part = warp_sum(part);
    __syncthreads();  // everyone has read red[] for f0
    if (lane == 0) red[warp] = part;
    __syncthreads();
    double rr = 0.0;
    for (int w = 0; w < NW; w++) rr += red[w];

    for (int m = 0; m < p.M; m++) {
        // ---- H1: each lane sums its task, one coalesced index load per step -------
        for (int rd = 0; rd < rounds; rd++) {
            const int steps = __ldg(wl + rd * NW + warp);  // warp-uniform
            if (steps == 0) continue;
            const PermT* pt = permt + __ldg(wb + rd * NW + warp) + lane;
            double acc = 0.0;
            for (int j = 0; j < steps; j += 4) {
                const uint32_t i0 = __ldg(pt + (j + 0) * 32), i1 = __ldg(pt + (j + 1) * 32);
                const uint32_t i2 = __ldg(pt + (j + 2) * 32), i3 = __ldg(pt + (j + 3) * 32);
                const double v0 = r[i0], v1 = r[i1], v2 = r[i2], v3 = r[i3];
                acc += v0; acc += v1; acc += v2; acc += v3;
            }
            const int dest = __ldg(tt_dest + rd * T + tid);
            if (dest >= 0) U[dest] = acc;
            else if (dest != kDiscard) pc[-dest - 1] = acc;
        }
        if (n_comb) {  // bins cut into pieces: combine in piece order
            __syncthreads();
            for (int c = tid; c < n_comb; c += T) {
                const int f = __ldg(comb_first + c), cnt = __ldg(comb_cnt + c);
                double v = pc[f];
                for (int q = 1; q < cnt; q++) v += pc[f + q];
                U[__ldg(comb_g + c)] = v;
            }
        }
        __syncthreads();
        // ---- H2-H4: one warp per learner, lane j = coefficient j -------------------
        for (int k = warp; k < K; k += NW) {
            // s_j = sum_l Zb[l][j] u[l] over the design points where B_j != 0
            double s0 = 0.0, s1 = 0.0;
            if (lane < d) {
                const int lb = __ldg(p.lwin + (k * d + lane) * 2), le = __ldg(p.lwin + (k * d + lane) * 2 + 1);
                const double* zc = p.Zb + (size_t)k * ns * d + lane;
                const double* u = U + k * ns;
                int l = lb;
                for (; l + 2 <= le; l += 2) {
                    s0 += __ldg(zc + (size_t)l * d) * u[l];
                    s1 += __ldg(zc + (size_t)(l + 1) * d) * u[l + 1];
                }
                if (l < le) s0 += __ldg(zc + (size_t)l * d) * u[l];
            }
            const double s = s0 + s1;
            // theta = A^-1 s (A^-1 symmetric: lane j reads column j of row j'), 4 chains
            const int jl = lane < d ? lane : 0;
            const double* Aj = p.Ainv + (size_t)k * d * d + jl;
            double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
            int jp = 0;
            for (; jp + 4 <= d; jp += 4) {
                const double a0 = __ldg(Aj + (jp + 0) * d), a1 = __ldg(Aj + (jp + 1) * d);
                const double a2 = __ldg(Aj + (jp + 2) * d), a3 = __ldg(Aj + (jp + 3) * d);
                t0 += a0 * __shfl_sync(0xffffffffu, s, jp + 0);
                t1 += a1 * __shfl_sync(0xffffffffu, s, jp + 1);
                t2 += a2 * __shfl_sync(0xffffffffu, s, jp + 2);
                t3 += a3 * __shfl_sync(0xffffffffu, s, jp + 3);
            }
            for (; jp < d; jp++) t0 += __ldg(Aj + jp * d) * __shfl_sync(0xffffffffu, s, jp);
            const double t = lane < d ? (t0 + t1) + (t2 + t3) : 0.0;
            // G theta on the band |j - j'| <= 3 (G is exactly banded)
            const double* Gk = p.G + (size_t)k * d * d;
            double gt = 0.0;
#pragma unroll
            for (int o = -(CWB_SPW - 1); o <= CWB_SPW - 1; o++) {
                const double to = __shfl_sync(0xffffffffu, t, (lane + o) & 31);
                const int jq = lane + o;
                if (lane < d && jq >= 0 && jq < d) gt += __ldg(Gk + jq * d + lane) * to;
            }
            double v = lane < d ? t * (2.0 * s - gt) : 0.0;
            v = warp_sum(v);
            th[k * 32 + lane] = t;
            if (lane == 0) delta[k] = v;
        }
        __syncthreads();
        // ---- H5: argmax delta (every thread, identical result) --------------------
        int ks = 0;
        double best = delta[0];
        for (int k = 1; k < K; k++) {
            const double v = delta[k];
            if (v > best) { best = v; ks = k; }
        }
        // ---- H6a: fitted values at the design points, aggregation, log ------------
        {
            const int32_t* j0 = p.zj0 + (size_t)ks * ns;
            const double* zs = p.Zs + (size_t)ks * ns * CWB_SPW;
            const double* tk = th + ks * 32;
            for (int l = tid; l < ns; l += T) {
                const int a = __ldg(j0 + l);
                double v = __ldg(zs + l * CWB_SPW) * tk[a];
#pragma unroll
                for (int q = 1; q < CWB_SPW; q++) v += __ldg(zs + l * CWB_SPW + q) * tk[a + q];
                zhat[l] = p.nu * v;
            }
            for (int j = tid; j < d; j += T) agg[ks * d + j] += p.nu * tk[j];
            if (tid == 0) {
                if (p.k_trace) p.k_trace[(size_t)m * p.B + b] = ks;
                if (p.sse_trace) p.sse_trace[(size_t)m * p.B + b] = rr - best;
            }
        }
        __syncthreads();
        // ---- H6b: residual update and r^T r ----------------------------------------
        {
            const IdxT* ik = idx + (size_t)ks * n;
            double acc = 0.0;
            for (int i = tid; i < n; i += T) {
                const double v = r[i] - zhat[__ldg(ik + i)];
                r[i] = v;
                acc += v * v;
            }
            acc = warp_sum(acc);
            if (lane == 0) red[warp] = acc;
            __syncthreads();
            rr = 0.0;
            for (int w = 0; w < NW; w++) rr += red[w];
            if (tid == 0 && p.risk_trace) p.risk_trace[(size_t)m * p.B + b] = rr / (2.0 * (double)n);
        }
        __syncthreads();  // red[] / r / zhat reuse in the next iteration
    }
    for (int a = tid; a < K * d; a += T) p.agg_out[(size_t)b * K * d + a] = agg[a];
    if (tid == 0 && p.offset_out) p.offset_out[b] = f0;
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

// One block.  Cuts every non-empty bin into ceil(count / P) tasks, sorts the
// tasks by length (descending, ties by bin order; coarse buckets), deals them
// to the T threads of the fused kernel in snake order and writes the row ids
// of every warp's 32 tasks step-major into permt.  Deterministic; runs once
// per data set inside cwb_init.
template <typename PermT, typename SrcPermT>
__global__ void k_fused_plan(const int32_t* __restrict__ off, const SrcPermT* __restrict__ perm, int K, int ns,
                             int n, int T, int P, size_t permt_cap, int32_t* __restrict__ plan,
                             int32_t* __restrict__ scratch, PermT* __restrict__ permt, const int* status) {
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
    for (int g = tid; g < KS; g += nthr) {
        const int k = g / ns, l = g - k * ns;
        const int c = off[k * (ns + 1) + l + 1] - off[k * (ns + 1) + l];
        const int pc = c > 0 ? (c + P - 1) / P : 0;
        pcs[g] = pc;
        first[g] = pc;
        slot[g] = pc > 1 ? pc : 0;
        cidx[g] = pc > 1 ? 1 : 0;
    }
    for (int e = tid; e < RM * T; e += nthr) tt_dest[e] = kDiscard;
    for (int e = tid; e < 2 * RM * NW; e += nthr) wl[e] = 0;
    for (size_t e = tid; e < permt_cap; e += nthr) permt[e] = (PermT)n;  // padding row
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
        if (pc > 1) {
            comb_g[cidx[g]] = g;
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
            s_dest[t] = pc == 1 ? g : -(slot[g] + q) - 1;
            const int bk = (int)(((long long)len * 1024) / (P + 1));
            s_bkt[t] = 1023 - min(1023, bk);  // ascending key = descending length
            st += len;
        }
    }
    __syncthreads();
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
                const int srt = (int)(hist[bk] + run_b[bk] + __popc(lt));
                const int rd = srt / T, i = srt - rd * T;
                const int th = (rd & 1) ? (T - 1 - i) : i;
                tt_dest[rd * T + th] = s_dest[t];
                s_slot[t] = rd * T + th;
                atomicMax(&wl[rd * NW + th / 32], (s_len[t] + 3) / 4 * 4);
            }
            __syncwarp();
            if (valid && lt == 0) run_b[bk] += __popc(mask);
            __syncwarp();
        }
    }
    __syncthreads();
    if (tid == 0) {  // block offsets, round count
        int o = 0, rounds = 0;
        for (int e = 0; e < RM * NW; e++) {
            wb[e] = o;
            o += 32 * wl[e];
            if (wl[e]) rounds = e / NW + 1;
        }
        plan[0] = n_tasks;
        plan[1] = rounds;
        plan[2] = n_comb;
        plan[3] = n_multi;
        plan[4] = P;
        plan[5] = o;
        plan[6] = plan[7] = 0;
    }
    __syncthreads();
    // row ids step-major; inside a task rows are ordered by shared-memory bank
    // pair (row mod 16) rotated by the lane, ties by bin-sorted position
    for (int t = tid; t < n_tasks; t += nthr) {
        const int sl = s_slot[t], rd = sl / T, thd = sl - rd * T, ln = thd & 31;
        PermT* out = permt + wb[rd * NW + thd / 32] + ln;
        const int st = s_start[t], len = s_len[t];
        int pos[16];
        for (int q = 0; q < 16; q++) pos[q] = 0;
        for (int q = 0; q < len; q++) pos[(((int)perm[st + q] & 15) - (ln & 15)) & 15]++;
        for (int q = 0, run = 0; q < 16; q++) { const int c = pos[q]; pos[q] = run; run += c; }
        for (int q = 0; q < len; q++) {  // stable counting sort by rotated bank pair
            const int row = (int)perm[st + q];
            out[(size_t)(pos[((row & 15) - (ln & 15)) & 15]++) * 32] = (PermT)row;
        }
    }
}

template <typename IdxT, typename PermT, int MAXT, int MINB>
int launch_t(const FusedParams& fp, size_t smem, cudaStream_t s) {
    auto kern = k_train_fused<IdxT, PermT, MAXT, MINB>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return -1;
    kern<<<fp.B, fp.T, smem, s>>>(fp);
    return 0;
}

template <typename IdxT, typename PermT>
int launch_sel(const FusedParams& fp, size_t smem, cudaStream_t s) {
    if (fp.T <= 384) return launch_t<IdxT, PermT, 384, 2>(fp, smem, s);
    return launch_t<IdxT, PermT, 768, 1>(fp, smem, s);
}

}  // namespace

static const size_t kMaxSmem = 227 * 1024;
static const size_t kTwoCtaSmem = 112 * 1024;

// Threads per CTA; false when the fused kernel cannot hold the working set.
static bool fused_shape(const cwb_ctx* c, int* T_out, size_t* smem_out) {
    if ((int64_t)c->K * c->n + 8 > INT32_MAX) return false;
    if ((int64_t)c->K * c->n_star * 16 > 200 * 1024) return false;  // plan kernel shared memory
    const int T_small = std::min(384, std::max(256, 32 * c->K));
    const int T_large = std::min(768, std::max(256, 32 * c->K));
    for (int pass = 0; pass < 2; pass++) {
        const int T = pass == 0 ? T_small : T_large;
        SmemLayout L((int)c->n, c->K, c->n_star, c->d, T, 2 * T);
        const size_t lim = pass == 0 ? kTwoCtaSmem : kMaxSmem;
        if (L.total <= lim) {
            *T_out = T;
            *smem_out = L.total;
            return true;
        }
    }
    return false;
}

size_t cwb_fused_smem_bytes(const cwb_ctx* c) {
    int T;
    size_t smem;
    return fused_shape(c, &T, &smem) ? smem : (size_t)-1;
}

int cwb_fused_plan(cwb_ctx* c, cudaStream_t s) {
    int T;
    size_t smem;
    c->fused_T = 0;
    if (!fused_shape(c, &T, &smem)) return CWB_OK;
    const int KS = c->K * c->n_star;
    const int total = (int)(c->K * c->n);
    const int P = std::max(4, (total + T - 1) / T);
    const size_t scratch_ints = 5 * (size_t)(KS + 2 * T);
    const size_t cap = permt_bound(KS, T, P);
    c->permt_bytes = c->n <= 65534 ? 2 : 4;
    if (cwb_alloc((void**)&c->plan, sizeof(int32_t) * (plan_ints(KS, T) + scratch_ints), s) != cudaSuccess ||
        cwb_alloc(&c->permt, (size_t)c->permt_bytes * cap, s) != cudaSuccess)
        return cwb_set_error(c, CWB_ENOMEM, "fused plan allocation failed");
    const size_t psmem = sizeof(int) * 4 * (size_t)KS;
    int32_t* scratch = c->plan + plan_ints(KS, T);
#define PLAN_CASE(PT, ST)                                                                              \
    {                                                                                                  \
        auto kern = k_fused_plan<PT, ST>;                                                              \
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem);           \
        kern<<<1, 1024, psmem, s>>>(c->off, (const ST*)c->perm, c->K, c->n_star, (int)c->n, T, P, cap, \
                                    c->plan, scratch, (PT*)c->permt, c->d_status);                      \
    }
    if (c->permt_bytes == 2 && c->perm_bytes == 2) PLAN_CASE(uint16_t, uint16_t)
    else if (c->permt_bytes == 2) PLAN_CASE(uint16_t, uint32_t)
    else if (c->perm_bytes == 2) PLAN_CASE(uint32_t, uint16_t)
    else PLAN_CASE(uint32_t, uint32_t)
#undef PLAN_CASE
    c->launches++;
    c->fused_T = T;
    c->fused_chunk = P;
    c->fused_smem = smem;
    return cwb_check_launch(c, "k_fused_plan");
}

int cwb_train_fused(cwb_ctx* c, const double* Y, int32_t B, double nu, int32_t M, double* offset_out,
                    double* theta_agg_out, int32_t* k_trace, double* sse_trace, double* risk_trace,
                    cudaStream_t s, bool* launched) {
    *launched = false;
    if (c->fused_T == 0) return CWB_OK;  // does not fit: caller uses the general path
    FusedParams fp;
    fp.n = (int)c->n; fp.K = c->K; fp.ns = c->n_star; fp.d = c->d; fp.M = M; fp.B = B; fp.nu = nu;
    fp.T = c->fused_T;
    fp.n_multi = 2 * c->fused_T;
    fp.Y = Y; fp.idx = c->idx; fp.permt = c->permt; fp.plan = c->plan; fp.zj0 = c->zj0; fp.Zs = c->Zs;
    fp.Zb = c->Zb; fp.lwin = c->lwin; fp.Ainv = c->Ainv; fp.G = c->G;
    fp.offset_out = offset_out; fp.agg_out = theta_agg_out;
    fp.k_trace = k_trace; fp.sse_trace = sse_trace; fp.risk_trace = risk_trace;
    fp.status = c->d_status;
    const size_t smem = c->fused_smem;
    int rc;
    const bool i8 = c->idx_bytes == 1, p16 = c->permt_bytes == 2;
    if (i8 && p16) rc = launch_sel<uint8_t, uint16_t>(fp, smem, s);
    else if (i8) rc = launch_sel<uint8_t, uint32_t>(fp, smem, s);
    else if (p16) rc = launch_sel<uint16_t, uint16_t>(fp, smem, s);
    else rc = launch_sel<uint16_t, uint32_t>(fp, smem, s);
    if (rc) return cwb_set_error(c, CWB_ECUDA, "fused kernel: cannot set shared memory size");
    c->launches++;
    *launched = true;
    return cwb_check_launch(c, "k_train_fused");
}
