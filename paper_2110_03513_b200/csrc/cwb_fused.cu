// cwb_fused.cu -- the whole CWB loop (Alg. 1 supp.) for one
// replication per CTA, all M iterations in one launch.
//
// Replications are independent boosting runs that share the binned pool, so
// a CTA never waits for another CTA: no grid barrier, no atomics, no host
// round trip between iterations.  The residual vector r (n doubles) and the
// bin sums u (K x n* doubles) stay in shared memory for all M iterations;
// the pool (bin inversion, sparse basis, cached inverse) is read-only and
// L1/L2 resident.  Per iteration m:
//
//   H1  u_k(l) = sum_{i in bin l of learner k} r_i      binMatVec loop
//       Threads take equal chunks of the K*n bin-sorted positions; a bin cut
//       by a chunk boundary is completed by a fixed-order carry pass.
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

#include "cwb_internal.cuh"

namespace {

struct FusedParams {
    int64_t n;
    int K, ns, d, M, B;
    double nu;
    int64_t chunk;  // bin-sorted positions per thread in H1
    const double* Y;
    const void* idx;
    const void* perm;
    const int32_t* off;
    const int32_t* zj0;
    const double* Zs;
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

template <typename T>
__host__ __device__ __forceinline__ size_t align16(size_t b) {
    return (b + 15) & ~(size_t)15;
}

struct SmemLayout {
    size_t r, U, th, delta, zhat, agg, carry, red, carry_bin, off, perm, total;
    __host__ __device__ SmemLayout(int64_t n, int K, int ns, int d, int T, int perm_bytes,
                                   bool perm_smem) {
        size_t o = 0;
        r = o; o = align16<char>(o + sizeof(double) * n);
        U = o; o = align16<char>(o + sizeof(double) * (size_t)K * ns);
        th = o; o = align16<char>(o + sizeof(double) * (size_t)K * 32);
        delta = o; o = align16<char>(o + sizeof(double) * K);
        zhat = o; o = align16<char>(o + sizeof(double) * ns);
        agg = o; o = align16<char>(o + sizeof(double) * (size_t)K * d);
        carry = o; o = align16<char>(o + sizeof(double) * T);
        red = o; o = align16<char>(o + sizeof(double) * 32);
        carry_bin = o; o = align16<char>(o + sizeof(int32_t) * T);
        off = o; o = align16<char>(o + sizeof(int32_t) * (size_t)K * (ns + 1));
        perm = o;
        if (perm_smem) o = align16<char>(o + (size_t)perm_bytes * K * n);
        total = o;
    }
};

template <typename IdxT, typename PermT, bool PERM_SMEM>
__global__ void __launch_bounds__(CWB_FUSED_THREADS, 2)
k_train_fused(FusedParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int T = CWB_FUSED_THREADS;
    constexpr int NW = T / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b = blockIdx.x;
    const int64_t n = p.n;
    const int K = p.K, ns = p.ns, d = p.d;
    const SmemLayout L(n, K, ns, d, T, (int)sizeof(PermT), PERM_SMEM);
    double* r = (double*)(smem + L.r);
    double* U = (double*)(smem + L.U);
    double* th = (double*)(smem + L.th);
    double* delta = (double*)(smem + L.delta);
    double* zhat = (double*)(smem + L.zhat);
    double* agg = (double*)(smem + L.agg);
    double* carry = (double*)(smem + L.carry);
    double* red = (double*)(smem + L.red);
    int32_t* carry_bin = (int32_t*)(smem + L.carry_bin);
    int32_t* off = (int32_t*)(smem + L.off);
    const PermT* perm = PERM_SMEM ? (const PermT*)(smem + L.perm) : (const PermT*)p.perm;
    const IdxT* idx = (const IdxT*)p.idx;

    // ---- I8: offset f0 = mean(y), r = y - f0, r^T r ------------------
    const double* y = p.Y + (size_t)b * n;
    double part = 0.0;
    bool bad = false;
    for (int64_t i = tid; i < n; i += T) {
        double v = y[i];
        bad |= !isfinite(v);
        r[i] = v;
        part += v;
    }
    if (bad) cwb_dev_fail(p.status, CWB_ENONFINITE);
    for (int a = tid; a < K * (ns + 1); a += T) off[a] = p.off[a];
    if (PERM_SMEM) {
        PermT* ps = (PermT*)(smem + L.perm);
        const PermT* pg = (const PermT*)p.perm;
        for (int64_t a = tid; a < (int64_t)K * n; a += T) ps[a] = pg[a];
    }
    for (int a = tid; a < K * d; a += T) agg[a] = 0.0;
    part = warp_sum(part);
    if (lane == 0) red[warp] = part;
    __syncthreads();
    double sy = 0.0;
    for (int w = 0; w < NW; w++) sy += red[w];
    const double f0 = sy / (double)n;
    part = 0.0;
    for (int64_t i = tid; i < n; i += T) {
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

    const int64_t total = (int64_t)K * n;
    const int64_t c = p.chunk;
    const int64_t p0 = (int64_t)tid * c;
    const int64_t p1 = p0 + c < total ? p0 + c : total;

    for (int m = 0; m < p.M; m++) {
        // ---- H1: bin sums over the bin-sorted positions [p0, p1) ----------------
        carry_bin[tid] = -1;
        if (p0 < p1) {
            int k = (int)(p0 / n);
            int64_t jloc = p0 - (int64_t)k * n;
            const int32_t* ok = off + k * (ns + 1);
            int lo = 0, hi = ns - 1;  // first l with off[l+1] > jloc
            while (lo < hi) {
                int mid = (lo + hi) >> 1;
                if (ok[mid + 1] > jloc) hi = mid;
                else lo = mid + 1;
            }
            int l = lo;
            int64_t base = (int64_t)k * n;
            int64_t bstart = base + ok[l], bend = base + ok[l + 1];
            double acc = 0.0;
            for (int64_t q = p0; q < p1; q++) {
                while (q >= bend) {
                    if (bstart < p0) { carry[tid] = acc; carry_bin[tid] = k * ns + l; }
                    else U[k * ns + l] = acc;
                    acc = 0.0;
                    if (++l == ns) { l = 0; k++; base += n; }
                    bstart = base + off[k * (ns + 1) + l];
                    bend = base + off[k * (ns + 1) + l + 1];
                }
                acc += r[perm[q]];
            }
            if (bstart < p0) { carry[tid] = acc; carry_bin[tid] = k * ns + l; }
            else U[k * ns + l] = acc;
        }
        __syncthreads();
        // carry pass: add the pieces of bins cut by chunk boundaries, in chunk order
        for (int g = tid; g < K * ns; g += T) {
            const int k = g / ns, l = g - k * ns;
            const int32_t a0 = off[k * (ns + 1) + l], a1 = off[k * (ns + 1) + l + 1];
            if (a1 == a0) { U[g] = 0.0; continue; }
            const int64_t s0 = (int64_t)k * n + a0, s1 = (int64_t)k * n + a1 - 1;
            const int64_t t0 = s0 / c, t1 = s1 / c;
            if (t1 > t0) {
                double v = U[g];
                for (int64_t t = t0 + 1; t <= t1; t++) v += carry[t];
                U[g] = v;
            }
        }
        __syncthreads();
        // ---- H2-H4: one warp per learner, lane j = coefficient j -----------------
        for (int k = warp; k < K; k += NW) {
            double s = 0.0;
            if (lane < d) {
                const int lb = p.lwin[(k * d + lane) * 2], le = p.lwin[(k * d + lane) * 2 + 1];
                const int32_t* j0 = p.zj0 + (size_t)k * ns;
                const double* zs = p.Zs + (size_t)k * ns * CWB_SPW;
                const double* u = U + k * ns;
                for (int l = lb; l < le; l++) s += zs[l * CWB_SPW + (lane - j0[l])] * u[l];
            }
            // theta = A^-1 s  (A^-1 symmetric: lane j reads column j of row j')
            const double* Ai = p.Ainv + (size_t)k * d * d;
            double t = 0.0;
            for (int jp = 0; jp < d; jp++) {
                double sj = __shfl_sync(0xffffffffu, s, jp);
                if (lane < d) t += Ai[jp * d + lane] * sj;
            }
            // G theta on the band |j - j'| <= 3 (G is exactly banded)
            const double* Gk = p.G + (size_t)k * d * d;
            double gt = 0.0;
#pragma unroll
            for (int o = -(CWB_SPW - 1); o <= CWB_SPW - 1; o++) {
                double to = __shfl_sync(0xffffffffu, t, (lane + o) & 31);
                int jp = lane + o;
                if (lane < d && jp >= 0 && jp < d) gt += Gk[jp * d + lane] * to;
            }
            double v = lane < d ? t * (2.0 * s - gt) : 0.0;
            v = warp_sum(v);
            th[k * 32 + lane] = lane < d ? t : 0.0;
            if (lane == 0) delta[k] = v;
        }
        __syncthreads();
        // ---- H5: argmax delta (every thread, identical result) ------------------
        int ks = 0;
        double best = delta[0];
        for (int k = 1; k < K; k++) {
            double v = delta[k];
            if (v > best) { best = v; ks = k; }
        }
        // ---- H6a: fitted values at the design points, aggregation, log ----------
        {
            const int32_t* j0 = p.zj0 + (size_t)ks * ns;
            const double* zs = p.Zs + (size_t)ks * ns * CWB_SPW;
            const double* tk = th + ks * 32;
            for (int l = tid; l < ns; l += T) {
                const int a = j0[l];
                double v = zs[l * CWB_SPW + 0] * tk[a];
#pragma unroll
                for (int q = 1; q < CWB_SPW; q++) v += zs[l * CWB_SPW + q] * tk[a + q];
                zhat[l] = p.nu * v;
            }
            for (int j = tid; j < d; j += T) agg[ks * d + j] += p.nu * tk[j];
            if (tid == 0) {
                if (p.k_trace) p.k_trace[(size_t)m * p.B + b] = ks;
                if (p.sse_trace) p.sse_trace[(size_t)m * p.B + b] = rr - best;
            }
        }
        __syncthreads();
        // ---- H6b: residual update and r^T r --------------------------------------
        {
            const IdxT* ik = idx + (size_t)ks * n;
            double acc = 0.0;
            for (int64_t i = tid; i < n; i += T) {
                double v = r[i] - zhat[ik[i]];
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

template <typename IdxT, typename PermT, bool PS>
int launch_t(const FusedParams& fp, size_t smem, cudaStream_t s) {
    auto kern = k_train_fused<IdxT, PermT, PS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return -1;
    kern<<<fp.B, CWB_FUSED_THREADS, smem, s>>>(fp);
    return 0;
}

}  // namespace

static const size_t kMaxSmem = 227 * 1024;
static const size_t kPermSmemBudget = 100 * 1024;

size_t cwb_fused_smem_bytes(const cwb_ctx* c, bool perm_in_smem) {
    SmemLayout L(c->n, c->K, c->n_star, c->d, CWB_FUSED_THREADS, c->perm_bytes, perm_in_smem);
    return L.total;
}

int cwb_train_fused(cwb_ctx* c, const double* Y, int32_t B, double nu, int32_t M, double* offset_out,
                    double* theta_agg_out, int32_t* k_trace, double* sse_trace, double* risk_trace,
                    cudaStream_t s, bool* launched) {
    *launched = false;
    size_t with_perm = cwb_fused_smem_bytes(c, true);
    size_t without = cwb_fused_smem_bytes(c, false);
    bool ps = with_perm <= kPermSmemBudget;
    size_t smem = ps ? with_perm : without;
    if (smem > kMaxSmem) return CWB_OK;  // does not fit: caller uses the general path
    FusedParams fp;
    fp.n = c->n; fp.K = c->K; fp.ns = c->n_star; fp.d = c->d; fp.M = M; fp.B = B; fp.nu = nu;
    int64_t total = (int64_t)c->K * c->n;
    fp.chunk = (total + CWB_FUSED_THREADS - 1) / CWB_FUSED_THREADS;
    fp.Y = Y; fp.idx = c->idx; fp.perm = c->perm; fp.off = c->off; fp.zj0 = c->zj0; fp.Zs = c->Zs;
    fp.lwin = c->lwin; fp.Ainv = c->Ainv; fp.G = c->G;
    fp.offset_out = offset_out; fp.agg_out = theta_agg_out;
    fp.k_trace = k_trace; fp.sse_trace = sse_trace; fp.risk_trace = risk_trace;
    fp.status = c->d_status;
    int rc;
    const bool i8 = c->idx_bytes == 1, p16 = c->perm_bytes == 2;
    if (i8 && p16) rc = ps ? launch_t<uint8_t, uint16_t, true>(fp, smem, s) : launch_t<uint8_t, uint16_t, false>(fp, smem, s);
    else if (i8) rc = ps ? launch_t<uint8_t, uint32_t, true>(fp, smem, s) : launch_t<uint8_t, uint32_t, false>(fp, smem, s);
    else if (p16) rc = ps ? launch_t<uint16_t, uint16_t, true>(fp, smem, s) : launch_t<uint16_t, uint16_t, false>(fp, smem, s);
    else rc = ps ? launch_t<uint16_t, uint32_t, true>(fp, smem, s) : launch_t<uint16_t, uint32_t, false>(fp, smem, s);
    if (rc) return cwb_set_error(c, CWB_ECUDA, "fused kernel: cannot set shared memory size");
    c->launches++;
    *launched = true;
    return cwb_check_launch(c, "k_train_fused");
}
