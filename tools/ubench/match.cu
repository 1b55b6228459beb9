// __match_any_sync latency / throughput on sm_100a (keys random in [0, nb)).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const unsigned* keys, int iters, unsigned* out, long long* cyc, int mode) {
    unsigned acc = 0, key = keys[threadIdx.x] + threadIdx.x * 2654435761u;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        unsigned m;
        if (mode == 0) m = __match_any_sync(0xffffffffu, key >> 22);      // throughput (independent)
        else m = __match_any_sync(0xffffffffu, (key >> 22) ^ (acc & 1));  // latency (dependent chain)
        acc += m;
        key = key * 1664525u + 1013904223u;  // per-lane sequences: 32 distinct 10-bit keys
        const unsigned k10 = key >> 22;
        acc ^= k10 << 1;
    }
    __syncthreads();
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    unsigned *keys, *out; long long* c;
    cudaMalloc(&keys, 4 * 1024); cudaMalloc(&out, 4 * 1024 * 148); cudaMalloc(&c, 8 * 148);
    cudaMemset(keys, 7, 4 * 1024);
    for (int mode = 0; mode < 2; mode++)
        for (int T : {32, 256, 512}) {
            const int iters = 4096;
            k<<<148, T>>>(keys, iters, out, c, mode);
            k<<<148, T>>>(keys, iters, out, c, mode);
            long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            printf("%s T=%d: %.1f cycles per warp-instruction per SM, %.1f cycles per iteration per warp\n",
                   mode ? "dependent" : "independent", T, (double)h / iters / (T / 32), (double)h / iters);
        }
}
