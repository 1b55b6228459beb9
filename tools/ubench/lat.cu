// Latency microbenchmarks on sm_100a: dependent chains, one warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, const double* g, int it) {
    __shared__ double sm[1024];
    double a = out[threadIdx.x], b = 1.0000001;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (double)(i % 7);
    __syncthreads();
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < it; i++) a = fma(a, b, 1e-9);
    t1 = clock64(); cyc[0] = t1 - t0;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < it; i++) a = a + b;
    t1 = clock64(); cyc[1] = t1 - t0;
    // SHFL double chain
    t0 = clock64();
    for (int i = 0; i < it; i++) a = __shfl_xor_sync(0xffffffffu, a, 1) + 0.0;
    t1 = clock64(); cyc[2] = t1 - t0;
    // LDS dependent chain (pointer chase through value)
    int j = threadIdx.x & 7;
    t0 = clock64();
    for (int i = 0; i < it; i++) { double v = sm[j]; j = ((int)v + i) & 1023; }
    t1 = clock64(); cyc[3] = t1 - t0;
    // DSETP + select chain
    t0 = clock64();
    for (int i = 0; i < it; i++) { double o = __shfl_xor_sync(0xffffffffu, a, 16); a = (o > a) ? o : a + 1.0; }
    t1 = clock64(); cyc[4] = t1 - t0;
    // LDG (L1 hit) dependent chain
    int q = threadIdx.x & 7;
    t0 = clock64();
    for (int i = 0; i < it; i++) { double v = __ldg(g + q); q = ((int)v + i) & 63; }
    t1 = clock64(); cyc[5] = t1 - t0;
    // DDIV
    t0 = clock64();
    for (int i = 0; i < it; i++) a = a / (2.0 * (double)(i + 3));
    t1 = clock64(); cyc[6] = t1 - t0;
    // BAR.SYNC (all threads)
    t0 = clock64();
    for (int i = 0; i < it; i++) __syncthreads();
    t1 = clock64(); cyc[7] = t1 - t0;
    out[threadIdx.x] = a + j + q;
}
int main() {
    double *o, *g; long long* c;
    cudaMalloc(&o, 8192); cudaMalloc(&g, 8192); cudaMalloc(&c, 64);
    cudaMemset(o, 0, 8192); cudaMemset(g, 0, 8192);
    const char* names[] = {"DFMA", "DADD", "SHFL.f64+DADD", "LDS chain", "SHFL+DSETP+sel", "LDG L1 chain", "DDIV", "BAR.SYNC(256t)"};
    for (int rep = 0; rep < 2; rep++) {
        k<<<1, 256>>>(o, c, g, 1000);
        long long h[8];
        cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
        if (rep) for (int i = 0; i < 8; i++) printf("%-18s %6.1f cycles\n", names[i], h[i] / 1000.0);
    }
    return 0;
}
