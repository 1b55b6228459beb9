// FP64 / on-chip peaks of this B200 for the roofline denominators of SURVEY Sec. 8(d)
// (VERDICT r1 "Next round" item 1): DADD and DFMA issue rate, L2 read bandwidth, HBM read
// bandwidth, shared-memory load bandwidth, and the TMEM load / store / read-modify-write rates
// (tcgen05.ld / tcgen05.st: TMEM as a lane-owned accumulator).
// DGEMM (the DMMA path) is measured by tools/peaks.py through cuBLAS.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench/peaks tools/ubench/peaks.cu
// Prints one JSON object per measurement on stdout.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

// ---------------------------------------------------------------- DADD / DFMA
template <int CH>
__global__ void k_dadd(double* out, int iters, double c) {
    double a[CH];
#pragma unroll
    for (int j = 0; j < CH; j++) a[j] = threadIdx.x * 1e-3 + j;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int j = 0; j < CH; j++) a[j] = __dadd_rn(a[j], c);
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < CH; j++) s += a[j];
    if (s == 12345.678) out[0] = s;
}

template <int CH>
__global__ void k_dfma(double* out, int iters, double b, double c) {
    double a[CH];
#pragma unroll
    for (int j = 0; j < CH; j++) a[j] = threadIdx.x * 1e-3 + j;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int j = 0; j < CH; j++) a[j] = __fma_rn(a[j], b, c);
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < CH; j++) s += a[j];
    if (s == 12345.678) out[0] = s;
}

// ---------------------------------------------------------------- global read bandwidth
__global__ void k_read(const double2* __restrict__ p, size_t n2, int passes, double* out) {
    double s0 = 0, s1 = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int ps = 0; ps < passes; ps++)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride * 4) {
            double2 v[4];
#pragma unroll
            for (int u = 0; u < 4; u++) v[u] = (i + u * stride < n2) ? __ldcg(p + i + u * stride) : make_double2(0, 0);
#pragma unroll
            for (int u = 0; u < 4; u++) { s0 += v[u].x; s1 += v[u].y; }
        }
    if (s0 + s1 == 12345.678) out[0] = s0;
}

// L2-resident gather-like read: every thread streams 8 independent 16-byte loads per step over a buffer that
// fits L2 (the access width of the wide H1 kernel); best of a few buffer sizes
__global__ void k_read8(const double2* __restrict__ p, size_t n2, int passes, double* out) {
    double s0 = 0, s1 = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const size_t per = n2 / 8;  // 8 independent streams
    for (int ps = 0; ps < passes; ps++)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < per; i += stride) {
            double2 v[8];
#pragma unroll
            for (int u = 0; u < 8; u++) v[u] = __ldcg(p + i + u * per);
#pragma unroll
            for (int u = 0; u < 8; u++) { s0 += v[u].x; s1 += v[u].y; }
        }
    if (s0 + s1 == 12345.678) out[0] = s0;
}

// ---------------------------------------------------------------- shared-memory loads
__global__ void k_lds(double* out, int iters, long long* cyc) {
    __shared__ __align__(16) double2 sm[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_double2(i, -i);
    __syncthreads();
    double s0 = 0, s1 = 0;
    int idx = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        const double2 v = sm[(idx + i * 32) & 2047];   // lane-contiguous: 32 x 16 B = 4 wavefronts
        s0 += v.x; s1 += v.y;
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (s0 + s1 == 12345.678) out[0] = s0;
}

// ---------------------------------------------------------------- TMEM
__device__ __forceinline__ uint32_t tmem_alloc512(uint32_t* slot) {
    if ((threadIdx.x >> 5) == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n"
                     :: "r"((uint32_t)__cvta_generic_to_shared(slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    return *slot;
}
__device__ __forceinline__ void tmem_free512(uint32_t a) {
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if ((threadIdx.x >> 5) == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" :: "r"(a));
}

// mode 0: loads only (x2 = 8 B per lane), 8 in flight per wait; 1: stores only;
// 2: fp64 read-modify-write of a warp-uniform column pair (the lane-owned accumulator pattern),
//    8 independent accumulators per wait (different column pairs)
__global__ void k_tmem(int mode, int iters, double* out, long long* cyc) {
    __shared__ uint32_t slot;
    const uint32_t base = tmem_alloc512(&slot);
    const int warp = threadIdx.x >> 5;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t cbase = (uint32_t)((warp >> 2) * 64);   // up to 8 warps share a quadrant -> distinct columns
    double acc = 0;
    const double v = 1.0 + threadIdx.x;
    const uint32_t vlo = (uint32_t)__double_as_longlong(v), vhi = (uint32_t)(__double_as_longlong(v) >> 32);
    // zero-initialise the columns used
    for (int c = 0; c < 16; c++) {
        const uint32_t a = base + lane_base + cbase + 2 * c;
        uint32_t z = 0;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n" :: "r"(a), "r"(z), "r"(z));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n");
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        if (mode == 0) {
            uint32_t r[16];
#pragma unroll
            for (int c = 0; c < 8; c++) {
                const uint32_t a = base + lane_base + cbase + 2 * ((c + i) & 15);
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];\n"
                             : "=r"(r[2 * c]), "=r"(r[2 * c + 1]) : "r"(a));
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int c = 0; c < 8; c++) acc += __longlong_as_double(((long long)r[2 * c + 1] << 32) | r[2 * c]);
        } else if (mode == 1) {
#pragma unroll
            for (int c = 0; c < 8; c++) {
                const uint32_t a = base + lane_base + cbase + 2 * ((c + i) & 15);
                asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n" :: "r"(a), "r"(vlo), "r"(vhi));
            }
        } else {
            uint32_t r[16];
#pragma unroll
            for (int c = 0; c < 8; c++) {
                const uint32_t a = base + lane_base + cbase + 2 * ((c * 2 + (i & 1)) & 15);
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];\n"
                             : "=r"(r[2 * c]), "=r"(r[2 * c + 1]) : "r"(a));
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int c = 0; c < 8; c++) {
                double x = __longlong_as_double(((long long)r[2 * c + 1] << 32) | r[2 * c]);
                x += v;
                const uint32_t a = base + lane_base + cbase + 2 * ((c * 2 + (i & 1)) & 15);
                asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n"
                             :: "r"(a), "r"((uint32_t)__double_as_longlong(x)),
                                "r"((uint32_t)(__double_as_longlong(x) >> 32)));
            }
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (mode == 2) {  // read back one accumulator so the RMW chain is live
        uint32_t lo, hi;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];\n" : "=r"(lo), "=r"(hi)
                     : "r"(base + lane_base + cbase));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        acc += __longlong_as_double(((long long)hi << 32) | lo);
    }
    if (acc == 12345.678) out[0] = acc;
    tmem_free512(base);
}

static float time_ms(cudaEvent_t a, cudaEvent_t b) { float ms; cudaEventElapsedTime(&ms, a, b); return ms; }

int main() {
    int dev = 0, sms = 0, clk_khz = 0;
    CK(cudaSetDevice(dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
    double* out; long long* cyc;
    CK(cudaMalloc(&out, 64)); CK(cudaMalloc(&cyc, 8 * 4096));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    printf("{\"what\": \"device\", \"sms\": %d, \"clock_rate_mhz\": %.0f}\n", sms, clk_khz / 1e3);

    // DADD / DFMA: 4 CTAs of 512 threads per SM, 8 independent chains per thread
    for (int fma = 0; fma < 2; fma++) {
        const int iters = 1 << 16, T = 512, G = sms * 4;
        for (int rep = 0; rep < 3; rep++) {
            cudaEventRecord(e0);
            if (fma) k_dfma<8><<<G, T>>>(out, iters, 0.9999999, 1e-9); else k_dadd<8><<<G, T>>>(out, iters, 1e-9);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            if (rep < 2) continue;
            const double ops = (double)G * T * iters * 8, s = time_ms(e0, e1) * 1e-3;
            printf("{\"what\": \"%s\", \"ops_per_s\": %.6g, \"per_sm_per_clk_at_max\": %.2f, \"ms\": %.3f, "
                   "\"note\": \"one %s per lane counted as one op\"}\n", fma ? "dfma" : "dadd", ops / s,
                   ops / s / sms / (clk_khz * 1e3), s * 1e3, fma ? "DFMA" : "DADD");
        }
    }
    CK(cudaGetLastError());

    // L2-resident read (32 MB, 40 passes) and HBM read (4 GiB, 2 passes)
    for (int which = 0; which < 2; which++) {
        const size_t bytes = which ? (size_t)4 << 30 : (size_t)32 << 20;
        const int passes = which ? 2 : 40;
        double2* p; CK(cudaMalloc(&p, bytes));
        CK(cudaMemset(p, 0, bytes));
        const size_t n2 = bytes / 16;
        float best = 1e30f;
        for (int rep = 0; rep < 5; rep++) {
            cudaEventRecord(e0);
            k_read<<<sms * 8, 512>>>(p, n2, passes, out);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            if (rep) best = fminf(best, time_ms(e0, e1));
        }
        printf("{\"what\": \"%s\", \"gb_per_s\": %.1f, \"bytes\": %zu, \"passes\": %d, \"ms\": %.3f}\n",
               which ? "hbm_read" : "l2_read", (double)bytes * passes / (best * 1e-3) / 1e9, bytes, passes, best);
        cudaFree(p);
    }
    CK(cudaGetLastError());

    // L2-resident reads, 8 x 16-byte loads in flight per thread
    for (size_t mb : {24, 48, 64, 96}) {
        const size_t bytes = mb << 20;
        double2* p; CK(cudaMalloc(&p, bytes));
        CK(cudaMemset(p, 0, bytes));
        float best = 1e30f;
        for (int T : {256, 512})
            for (int occ : {4, 8}) {
                for (int rep = 0; rep < 4; rep++) {
                    cudaEventRecord(e0);
                    k_read8<<<sms * occ, T>>>(p, bytes / 16, 20, out);
                    cudaEventRecord(e1);
                    CK(cudaEventSynchronize(e1));
                    if (rep) best = fminf(best, time_ms(e0, e1));
                }
            }
        printf("{\"what\": \"l2_read8_%zuMB\", \"gb_per_s\": %.1f, \"bytes\": %zu, \"passes\": 20, \"ms\": %.3f}\n", mb,
               (double)bytes * 20 / (best * 1e-3) / 1e9, bytes, best);
        cudaFree(p);
    }
    // shared memory LDS.128
    {
        const int iters = 1 << 14;
        for (int T : {256, 512, 1024}) {
            k_lds<<<sms, T>>>(out, iters, cyc);
            CK(cudaDeviceSynchronize());
            long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("{\"what\": \"smem_lds128\", \"threads\": %d, \"bytes_per_clk_per_sm\": %.1f}\n", T,
                   (double)T * iters * 16 / c);
        }
    }
    // TMEM: loads, stores, fp64 read-modify-write
    {
        const int iters = 1 << 12;
        const char* names[3] = {"tmem_ld_32x32b_x2", "tmem_st_32x32b_x2", "tmem_rmw_f64"};
        for (int mode = 0; mode < 3; mode++)
            for (int T : {128, 256, 512}) {
                k_tmem<<<sms, T>>>(mode, iters, out, cyc);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("{\"what\": \"%s\", \"error\": \"%s\"}\n", names[mode], cudaGetErrorString(e)); return 1; }
                long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
                const double lane_ops = (double)T * iters * 8;   // 8-byte lane accesses (RMW: one per add)
                printf("{\"what\": \"%s\", \"threads\": %d, \"lane_ops_per_clk_per_sm\": %.2f, \"bytes_per_clk_per_sm\": %.1f}\n",
                       names[mode], T, lane_ops / c, lane_ops * 8 / c);
            }
    }
    return 0;
}
