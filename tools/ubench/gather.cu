// Shared-memory gather throughput on sm_100a: each lane sums doubles (RB=1) or double2
// (RB=2) at byte offsets read from a u16 schedule in shared memory, groups of 4 steps.
// conflict-free schedule (distinct bank groups per wavefront) vs random.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
template <int RB, int UNR>
__global__ void k(const uint16_t* sched_g, int steps, int rows, double* out, long long* cyc) {
    extern __shared__ __align__(16) unsigned char sm[];
    double* r = (double*)sm;
    uint16_t* sched = (uint16_t*)(sm + 16 * (rows + 16));
    const int T = blockDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < RB * (rows + 16); i += T) r[i] = 1.0 + (i & 7);
    const int per_warp = steps * 32;
    for (int i = tid; i < per_warp * (T / 32); i += T) sched[i] = sched_g[i];
    __syncthreads();
    const uint16_t* pt = sched + warp * per_warp + lane * 4;
    double a0 = 0, a1 = 0, b0 = 0, b1 = 0;
    long long t0 = clock64();
    for (int rep = 0; rep < 20; rep++) {
#pragma unroll UNR
        for (int j = 0; j < steps; j += 4) {
            const uint2 v = *reinterpret_cast<const uint2*>(pt + j * 32);
            const uint32_t o[4] = {v.x & 0xffffu, v.x >> 16, v.y & 0xffffu, v.y >> 16};
#pragma unroll
            for (int e = 0; e < 4; e++) {
                if (RB == 2) {
                    const double2 x = *reinterpret_cast<const double2*>(sm + o[e]);
                    if (e & 1) { a1 += x.x; b1 += x.y; } else { a0 += x.x; b0 += x.y; }
                } else {
                    const double x = *reinterpret_cast<const double*>(sm + o[e]);
                    if (e & 1) a1 += x; else a0 += x;
                }
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    out[blockIdx.x * T + tid] = a0 + a1 + b0 + b1;
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    const int rows = 1331, steps = 64;
    for (int RB = 1; RB <= 2; RB++)
    for (int T : {256, 512, 1024})
    for (int mode = 0; mode < 2; mode++) {
        const int NW = T / 32, G = 16 / RB;
        uint16_t* h = (uint16_t*)malloc(2 * steps * 32 * NW);
        srand(1);
        for (int w = 0; w < NW; w++)
            for (int s = 0; s < steps; s++)
                for (int ln = 0; ln < 32; ln++) {
                    int row;
                    if (mode == 0) {  // conflict-free: lane group slot -> distinct colour
                        int c = ((ln % G) + s) % G;
                        row = (rand() % (rows / G)) * G + c;
                    } else row = rand() % rows;
                    h[w * steps * 32 + (s / 4) * 128 + ln * 4 + (s % 4)] = (uint16_t)(row * 8 * RB);
                }
        uint16_t* d; double* o; long long* c;
        cudaMalloc(&d, 2 * steps * 32 * NW); cudaMalloc(&o, 8 * 148 * 1024); cudaMalloc(&c, 8 * 148);
        cudaMemcpy(d, h, 2 * steps * 32 * NW, cudaMemcpyHostToDevice);
        size_t smem = 16 * (rows + 16) + 2 * steps * 32 * NW;
        long long hc[148];
        if (RB == 1) { cudaFuncSetAttribute(k<1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); k<1, 4><<<148, T, smem>>>(d, steps, rows, o, c); k<1, 4><<<148, T, smem>>>(d, steps, rows, o, c); }
        else { cudaFuncSetAttribute(k<2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); k<2, 4><<<148, T, smem>>>(d, steps, rows, o, c); k<2, 4><<<148, T, smem>>>(d, steps, rows, o, c); }
        cudaDeviceSynchronize();
        cudaMemcpy(hc, c, 8 * 148, cudaMemcpyDeviceToHost);
        const double lanes_loads = 20.0 * steps * T;  // lane-loads per CTA
        printf("RB=%d T=%4d %-13s cycles %8lld  bytes/clk %.1f  lane-loads/clk %.2f  err=%s\n", RB, T,
               mode ? "random" : "conflict-free", hc[0], lanes_loads * 8 * RB / hc[0], lanes_loads / hc[0],
               cudaGetErrorString(cudaGetLastError()));
        cudaFree(d); cudaFree(o); cudaFree(c); free(h);
    }
}
