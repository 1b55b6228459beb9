// Shared-memory atomic add throughput on B200 (lane-ops per clock per SM), for the B = 1 findBest design question:
// can a row-streaming weighted histogram with integer (fixed-point limb) shared-memory atomics keep up with HBM?
// Modes: u32 / u64 atomicAdd with distinct addresses per lane (bank-spread) and with pseudo-random bins of a
// 1000-bin histogram per warp (the R4 shape), result unused (RED) or used.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o atoms atoms.cu ; run: ./atoms
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int T = 1024, ITER = 4096;

template <typename V, int MODE>
__global__ void __launch_bounds__(T, 1) k_atoms(unsigned long long* out, long long* cyc) {
    extern __shared__ unsigned char sm[];
    V* h = (V*)sm;                      // 32 warps x 1024 bins (8-byte types: two warps share one)
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    constexpr int SH = sizeof(V) / 4;
    V* hw = h + (w / SH) * 1024;
    for (int i = tid; i < 32 / SH * 1024; i += T) h[i] = 0;
    __syncthreads();
    uint32_t x = 2654435761u * (tid + 1) + blockIdx.x;
    const long long t0 = clock64();
    V acc = 0;
#pragma unroll 8
    for (int i = 0; i < ITER; i++) {
        int a;
        x = x * 1664525u + 1013904223u;
        if (MODE == 0) a = (lane * 33 + i * 7) & 1023;   // distinct bank per lane
        else a = (x >> 8) % 1000;  // random bins of a 1000-bin histogram
        const V v = (V)((x >> 3) & 0xff) + (V)i;  // a data-dependent addend (a constant 1 becomes ATOMS.POPC.INC)
        if (MODE == 2) acc += atomicAdd(&hw[a], v);   // result used
        else atomicAdd(&hw[a], v);
    }
    __syncthreads();
    const long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
    if (acc == (V)12345) out[0] = 1;
    if (tid == 0) out[1 + blockIdx.x] = (unsigned long long)hw[5];
}

template <typename V, int MODE>
void run(const char* name, int nsm) {
    unsigned long long* out;
    long long* cyc;
    cudaMalloc(&out, 8 * (nsm + 1));
    cudaMalloc(&cyc, 8 * nsm);
    const int smem = 32 / (sizeof(V) / 4) * 1024 * sizeof(V);
    cudaFuncSetAttribute(k_atoms<V, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_atoms<V, MODE><<<nsm, T, smem>>>(out, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_atoms<V, MODE><<<nsm, T, smem>>>(out, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c[1];
    cudaMemcpy(c, cyc, 8, cudaMemcpyDeviceToHost);
    const double ops = (double)T * ITER;  // per SM
    printf("%-34s %6.2f lane-ops/clk/SM (CTA 0: %lld cycles), %.1f G ops/s total, %.3f ms\n", name, ops / c[0], c[0],
           ops * nsm / (ms * 1e6), ms);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    int dev = 0, nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    run<unsigned int, 0>("u32 atomicAdd, bank-spread", nsm);
    run<unsigned int, 1>("u32 atomicAdd, random of 1000 bins", nsm);
    run<unsigned int, 2>("u32 atomicAdd, random, result used", nsm);
    run<unsigned long long, 0>("u64 atomicAdd, bank-spread", nsm);
    run<unsigned long long, 1>("u64 atomicAdd, random of 1000 bins", nsm);
    run<double, 1>("f64 atomicAdd, random of 1000 bins", nsm);
    return 0;
}
