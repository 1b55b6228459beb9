// cwb_stream.cu -- streaming binMatVec (H1) for a few residual vectors
// over large n: the index-streaming path of findBestBaselearner (SURVEY Sec. 8(d)
// target: one residual column at R3/R4 sizes, bound by HBM on the index stream).
//
// binMatVec for learner k is u_k(l) = sum_{i : idx_k(i) = l} r_i.  On
// B200 the scatter-add of the paper's loop would be an fp64 shared-memory atomic (a
// CAS loop on sm_100a); instead the bins are inverted per chunk of rows once per pool
// (the "hash map" of P:L861, stored as a gather plan) and every lane *gathers* the
// rows of one bin into a register:
//
//   plan (built once, lazily, on the first narrow findBest):
//     rows are cut into chunks of C = 8176 (a chunk of r is ~64 KB of shared memory);
//     learners into groups of Ks (the group's bin sums, Ks * n* doubles, stay in
//     shared memory across chunks).  For every item (learner group, chunk) the
//     non-empty bins of the group's learners are tasks; tasks are sorted by row count
//     (descending) and dealt to lanes 32 at a time, so the 32 lanes of a warp-group
//     sum bins of (nearly) equal length.  Entries are chunk-local row ids (u16) laid
//     out [step/4][lane][4]: one coalesced 8-byte load per lane per 4 steps.  Lanes
//     past their bin's end read padding rows C + (lane mod 16) (zeros, distinct banks).
//   kernel k_h1_stream: CTA = (learner group, contiguous chunk range, column q).  Per
//     chunk: the residual chunk is loaded into shared memory, every warp takes groups
//     of the item round-robin, gathers r[row] from shared memory and adds, and the
//     lane adds its bin total into the CTA's bin sums (each (learner, bin) is one task
//     per item: no conflicting writes).  At the end the CTA writes its bin sums; a
//     combine kernel adds the CTA partials of a learner group in CTA order.
//
// Deterministic: every sum has a fixed order (plan order within a bin and chunk,
// chunks ascending within a CTA, CTAs ascending in the combine).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "cwb_internal.cuh"

namespace {

#ifndef CWB_STREAM_KC
#define CWB_STREAM_KC 8176
#endif
constexpr int kC = CWB_STREAM_KC;  // rows per chunk: byte offsets of rows and pad rows (C..C+15) fit u16
constexpr int kPad = 16;        // zero padding rows after the chunk
constexpr int kUBudget = 7168;  // doubles of bin sums per CTA (56 KB): Ks * n* <= kUBudget
constexpr int kStreamT = 1024;  // threads of the stream kernel (one CTA per SM)
constexpr int kNWK = kStreamT / 32;  // kernel warps: the plan deals groups to them
constexpr int kStage = 4;        // entry blocks per register stage (two stages in flight per warp)
constexpr int kFitSplitMax = 8;  // threads per bin sum in k_fit_narrow's combine

// ---------------------------------------------------------------- plan kernels
// bin counts of every (learner, chunk): cnt[(k * nch + c) * ns + l]
template <typename IdxT>
__global__ void k_sp_count(const IdxT* __restrict__ idx, int64_t n, int ns, int nch, uint32_t* __restrict__ cnt) {
    extern __shared__ uint32_t h[];
    const int c = blockIdx.x, k = blockIdx.y;
    for (int l = threadIdx.x; l < ns; l += blockDim.x) h[l] = 0;
    __syncthreads();
    const int64_t r0 = (int64_t)c * kC, r1 = min(n, r0 + kC);
    const IdxT* ik = idx + (size_t)k * n;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) atomicAdd(&h[ik[i]], 1u);
    __syncthreads();
    uint32_t* o = cnt + ((size_t)k * nch + c) * ns;
    for (int l = threadIdx.x; l < ns; l += blockDim.x) o[l] = h[l];
}

// start of chunk c's rows inside bin l of the bin inversion (perm is ascending within a bin)
__global__ void k_sp_start(const uint32_t* __restrict__ cnt, const int32_t* __restrict__ off, int K, int ns,
                           int nch, uint32_t* __restrict__ cst) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= (int64_t)K * ns) return;
    const int k = (int)(g / ns), l = (int)(g - (int64_t)k * ns);
    uint32_t run = (uint32_t)off[(size_t)k * (ns + 1) + l];
    for (int c = 0; c < nch; c++) {
        const size_t e = ((size_t)k * nch + c) * ns + l;
        cst[e] = run;
        run += cnt[e];
    }
}

// One block per item (learner group lg, chunk c): sort the group's non-empty bins by
// count (descending, ties by task id) with a bitonic sort of packed keys in shared
// memory; write the sorted task ids (kl * ns + l) and the item's group / block counts.
__global__ void k_sp_sort(const uint32_t* __restrict__ cnt, int K, int ns, int nch, int Ks, int NTP,
                          uint32_t* __restrict__ tasks, int2* __restrict__ isize) {
    extern __shared__ unsigned long long key[];
    const int item = blockIdx.x, lg = item / nch, c = item - lg * nch;
    const int k0 = lg * Ks, ke = min(K, k0 + Ks), NT = (ke - k0) * ns;
    for (int t = threadIdx.x; t < NTP; t += blockDim.x) {
        unsigned long long v = ~0ull;
        if (t < NT) {
            const int kl = t / ns, l = t - kl * ns;
            const uint32_t q = cnt[((size_t)(k0 + kl) * nch + c) * ns + l];
            if (q) v = ((unsigned long long)(0xffffffffu - q) << 32) | (uint32_t)t;
        }
        key[t] = v;
    }
    __syncthreads();
    for (int size = 2; size <= NTP; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < NTP / 2; t += blockDim.x) {
                const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const unsigned long long a = key[lo], b = key[hi];
                if ((a > b) == up) { key[lo] = b; key[hi] = a; }
            }
            __syncthreads();
        }
    __shared__ int s_nt;
    if (threadIdx.x == 0) s_nt = 0;
    __syncthreads();
    uint32_t* tk = tasks + (size_t)item * NTP;
    for (int t = threadIdx.x; t < NTP; t += blockDim.x) {
        const unsigned long long v = key[t];
        tk[t] = v == ~0ull ? 0xffffffffu : (uint32_t)v;
        if (v != ~0ull && (t + 1 == NTP || key[t + 1] == ~0ull)) s_nt = t + 1;
    }
    __syncthreads();
    if (threadIdx.x == 0) isize[item] = make_int2((s_nt + 31) / 32, 0);  // blocks: k_sp_sched<false>
}

// exclusive scan of the (groups, blocks) counts of the items (one thread: items <= a few thousand)
__global__ void k_sp_scan(const int2* __restrict__ isize, int nitems, int2* __restrict__ ibase,
                          long long* __restrict__ tot) {
    long long g = 0, b = 0;
    for (int i = 0; i < nitems; i++) {
        ibase[i] = make_int2((int)g, (int)b);
        g += isize[i].x;
        b += isize[i].y;
    }
    tot[0] = g;
    tot[1] = b;
}

// Gather schedule of one item: one block per item, one warp per 32-task group.  The 16
// lanes of a half-warp read 8-byte rows in one shared-memory wavefront when the rows
// have distinct colours (row mod 16 = bank pair).  Every step each half-warp assigns
// colours greedily: the lane with the most rows left picks first (ties: lowest lane),
// taking the free colour it holds most rows of; lanes without a pick read padding
// rows C + (a free colour), so every step is conflict-free.  Steps run until the
// warp's 32 bins are exhausted, rounded up to a multiple of 4 with padding steps.
// EMIT = false: count the steps (isize[item].y += blocks); EMIT = true: write entries,
// group table and destinations at the scanned offsets.
// kernel warp of group g (the stream kernel deals the groups of an item to its kNWK warps in snake
// order: round g / kNWK left to right when even, right to left when odd) and the warp-major order key
__device__ __forceinline__ int gwarp(int g) {
    const int r = g / kNWK, x = g - r * kNWK;
    return (r & 1) ? kNWK - 1 - x : x;
}
__device__ __forceinline__ uint32_t gorder(int g) { return ((uint32_t)gwarp(g) << 16) | (uint32_t)(g / kNWK); }

// first entry block of every kernel warp's stream in item `item` (+ the item's end)
__global__ void k_sp_wstart(const int2* __restrict__ isize, const int2* __restrict__ ibase,
                            const uint32_t* __restrict__ gsteps, int NTP, uint32_t* __restrict__ wst) {
    const int item = blockIdx.x, lane = threadIdx.x;  // lane = kernel warp
    const int ng = isize[item].x;
    const uint32_t* gs = gsteps + (size_t)item * (NTP / 32);
    if (lane < kNWK) {
        uint32_t part = 0;
        for (int h = 0; h < ng; h++) part += gwarp(h) < lane ? gs[h] / 4 : 0u;
        wst[(size_t)item * (kNWK + 1) + lane] = (uint32_t)ibase[item].y + part;
    }
    if (lane == 0) wst[(size_t)item * (kNWK + 1) + kNWK] = (uint32_t)(ibase[item].y + isize[item].y);
}

template <typename PermT, bool EMIT>
__global__ void __launch_bounds__(512) k_sp_sched(
    const uint32_t* __restrict__ tasks, const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ cst,
    const PermT* __restrict__ perm, int64_t n, int ns, int nch, int Ks, int NTP, int2* __restrict__ isize,
    const int2* __restrict__ ibase, uint32_t* __restrict__ gsteps, uint16_t* __restrict__ ent,
    uint2* __restrict__ gtab, uint16_t* __restrict__ dest) {
    const int item = blockIdx.x, lg = item / nch, c = item - lg * nch;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int hl = lane & 15, hb = lane & 16;
    const unsigned hmask = 0xffffu << hb;
    const int ng = isize[item].x;
    const uint32_t* tk = tasks + (size_t)item * NTP;
    uint32_t* gs = gsteps + (size_t)item * (NTP / 32);
    const uint32_t base = (uint32_t)c * kC;
    for (int g = w; g < ng; g += nw) {
        const uint32_t t = tk[32 * g + lane];
        int rem = 0;
        uint32_t st = 0;
        int k = lg * Ks;
        if (t != 0xffffffffu) {
            const uint32_t kl = t / ns, l = t - kl * ns;
            k += (int)kl;
            const size_t e = ((size_t)k * nch + c) * ns + l;
            rem = (int)cnt[e];
            st = cst[e];
        }
        const PermT* rows = perm + (size_t)k * n + st;
        int cc[16], pos[16];
#pragma unroll
        for (int x = 0; x < 16; x++) { cc[x] = 0; pos[x] = 0; }
        for (int s = 0; s < rem; s++) cc[((uint32_t)rows[s] - base) & 15]++;
        uint16_t* eg = nullptr;
        uint32_t nblk_g = 0;
        if (EMIT) {
            // blocks in warp-major order: the groups of kernel warp 0 (snake-dealt, see gwarp), then of
            // warp 1, ...; within a warp in dealing order
            const uint32_t og = gorder(g);
            uint32_t part = 0;
            for (int h = lane; h < ng; h += 32) part += gorder(h) < og ? gs[h] / 4 : 0u;
            for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            const uint32_t bb = (uint32_t)ibase[item].y + part;
            nblk_g = gs[g] / 4;
            const int gg = ibase[item].x + g;
            if (lane == 0) gtab[gg] = make_uint2(bb, gs[g] / 4);
            dest[(size_t)gg * 32 + lane] = t != 0xffffffffu ? (uint16_t)t : (uint16_t)0xffff;
            eg = ent + (size_t)bb * 128 + lane * 4;
        }
        uint32_t steps = 0;
        while (__any_sync(0xffffffffu, rem > 0) || (steps & 3)) {
            // colours used once (fr2) may take a second lane (a 2-way conflict: one extra wavefront)
            // rather than leave the lane a padding entry: the entry stream, not the shared-memory pipe,
            // is the bound of the stream kernel
            unsigned fr = 0xffffu, fr2 = 0u;
            int pick = -1;
            bool assigned = false;
            for (int r = 0; r < 16; r++) {
                int key = assigned ? -1 : ((rem << 4) | (15 - hl));
#pragma unroll
                for (int o = 8; o; o >>= 1) key = max(key, __shfl_xor_sync(hmask, key, o));
                if (key < 16) break;  // the best unassigned lane has no rows left: the rest pad
                const int win = 15 - (key & 15);
                int x = -1;
                if (hl == win) {
                    int best = 0;
#pragma unroll
                    for (int y = 0; y < 16; y++)
                        if (((fr >> y) & 1u) && cc[y] > best) { best = cc[y]; x = y; }
                    if (x < 0) {
                        best = 0;
#pragma unroll
                        for (int y = 0; y < 16; y++)
                            if (((fr2 >> y) & 1u) && cc[y] > best) { best = cc[y]; x = y; }
                    }
                    assigned = true;
                    pick = x;
                }
                x = __shfl_sync(hmask, x, hb | win);
                if (x >= 0) {
                    if ((fr >> x) & 1u) { fr &= ~(1u << x); fr2 |= 1u << x; }
                    else fr2 &= ~(1u << x);
                }
            }
            const unsigned np = (~__ballot_sync(0xffffffffu, pick >= 0) >> hb) & 0xffffu;  // lanes padding
            uint16_t v;
            if (pick >= 0) {
                int p = pos[pick];
                while ((((uint32_t)rows[p] - base) & 15) != (uint32_t)pick) p++;
                v = (uint16_t)(((uint32_t)rows[p] - base) * 8u);  // byte offset in the staged chunk
                pos[pick] = p + 1;
                cc[pick]--;
                rem--;
            } else {  // padding row of a free colour, else of a colour used once, else any
                int rank = __popc(np & ((1u << hl) - 1u));
                const int n1 = __popc(fr), n2 = __popc(fr2);
                unsigned f = rank < n1 ? fr : (rank < n1 + n2 ? fr2 : 0xffffu);
                rank = rank < n1 ? rank : (rank < n1 + n2 ? rank - n1 : (rank - n1 - n2) & 15);
                while (rank--) f &= f - 1u;
                v = (uint16_t)((kC + (__ffs(f) - 1)) * 8);
            }
            // bit 0 (free: byte offsets of 8-byte rows) of the first entry of the group's last block of
            // every lane: the kernel flushes the lane's bin total after that block
            if (EMIT && (steps >> 2) + 1 == nblk_g && (steps & 3) == 0) v |= 1;
            if (EMIT) eg[(size_t)(steps >> 2) * 128 + (steps & 3)] = v;
            steps++;
        }
        if (!EMIT && lane == 0) {
            gs[g] = steps;
            atomicAdd(&isize[item].y, (int)(steps / 4));
        }
    }
}

// ---------------------------------------------------------------- stream kernel
// grid (N, B), two CTAs per SM: CTA j takes the items [j I / N, (j+1) I / N) of the (learner
// group major, chunk minor) item order, column q = blockIdx.y.  When the learner group
// changes, the bin sums go to the CTA's next partial slot P[q][j][slot] (slot = lg - first
// lg of j).  Per item the residual chunk, the group table and the destinations are staged in
// shared memory.  Each warp streams the entry blocks of its groups (groups w, w + nw, ...)
// as pieces of kPiece blocks through registers, two pieces ahead of the gathers.  Entries
// are byte offsets of rows in the staged chunk (LDS [R + UR]).
constexpr int kPiece = 4;      // entry blocks (256 B) per piece
constexpr int kMaxG = kUBudget / 32;  // groups per item staged in shared memory (Ks * n* <= kUBudget)

__device__ __forceinline__ double gat(const unsigned char* __restrict__ rb, uint32_t off) {
    return *(const double*)(rb + off);
}
__device__ __forceinline__ double gather4(const unsigned char* __restrict__ rb, uint2 v) {
    // fixed order: entries 0, 1, 2, 3 of the block
    double a = gat(rb, v.x & 0xfffe);  // bit 0 of entry 0: end-of-group flag
    a += gat(rb, v.x >> 16);
    a += gat(rb, v.y & 0xffff);
    a += gat(rb, v.y >> 16);
    return a;
}

struct Piece {
    uint2 v[kPiece];
};

__device__ __forceinline__ uint32_t sm_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            sm_u32(bar)),
        "r"(parity)
        : "memory");
}
// TMA bulk copy global -> shared, completion counted on an mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sm_u32(dst)),
                 "l"(src), "r"(bytes), "r"(sm_u32(bar))
                 : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async(void* dst, const void* src) {
    if (N == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sm_u32(dst)), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(sm_u32(dst)), "l"(src), "n"(N) : "memory");
}
__device__ __forceinline__ void cp_async_commit_wait_all() {
    asm volatile("cp.async.commit_group;\n cp.async.wait_all;" ::: "memory");
}

// One CTA per SM (kStreamT threads).  The chunk of residuals and the group tables of item
// it + 1 are copied into the second buffer (TMA bulk copy for the chunk, cp.async for the tables)
// while item it is gathered, so the copies overlap the gathers.
__global__ void __launch_bounds__(kStreamT, 1)
    k_h1_stream(const double* __restrict__ R, int64_t n, int nch, int Ks, int ns, int nitems, int nslot,
                const uint2* __restrict__ ent, const uint2* __restrict__ gtab, const uint16_t* __restrict__ dest,
                const int2* __restrict__ isize, const int2* __restrict__ ibase, const uint32_t* __restrict__ wst,
                double* __restrict__ P, double* __restrict__ rrp, int* status) {
    extern __shared__ __align__(16) double sm[];
    __shared__ double red[kStreamT / 32];
    __shared__ __align__(16) uint32_t s_ws[2][kNWK + 4];
    __shared__ __align__(16) uint16_t s_dst[2][kMaxG * 32];
    __shared__ __align__(8) uint64_t bars[2];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
    const int NU = Ks * ns;
    // two chunk buffers sm + bf (kC + kPad): kC residuals + kPad zero rows each
    double* U = sm + 2 * (kC + kPad);                // Ks * ns bin sums
    const int N = gridDim.x, j = blockIdx.x, q = blockIdx.y;
    const int i0 = (int)((int64_t)nitems * j / N), i1 = (int)((int64_t)nitems * (j + 1) / N);
    double* Pj = P + ((size_t)q * N + j) * nslot * NU;
    const double* col = R + (size_t)q * n;
    const bool tma = (((uintptr_t)col) & 15) == 0;   // chunk starts are 16-byte aligned iff the column is
    // programmatic dependent launch: k_fit_narrow may start its prologue on SMs this grid frees
    // (it waits for this grid's completion before it reads P and rrp)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    for (int a = tid; a < NU; a += blockDim.x) U[a] = 0.0;
    if (tid < 2 * kPad) sm[(tid / kPad) * (kC + kPad) + kC + (tid % kPad)] = 0.0;
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // copies of item it into buffer bf: chunk (TMA, tail row and unaligned columns by plain loads),
    // group table and destinations (cp.async)
    auto issue = [&](int it, int bf) {
        const int lg = it / nch, c = it - lg * nch;
        const int64_t r0 = (int64_t)c * kC;
        const int len = (int)min((int64_t)kC, n - r0);
        double* rs = sm + bf * (kC + kPad);
        if (tma) {
            if (tid == 0) {
                const uint32_t bytes = (uint32_t)((size_t)len * 8) & ~15u;
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&bars[bf], bytes);
                if (bytes) bulk_g2s(rs, col + r0, bytes, &bars[bf]);
                if (len & 1) rs[len - 1] = __ldg(col + r0 + len - 1);
            }
        } else {
            for (int i = tid; i < len; i += blockDim.x) rs[i] = __ldg(col + r0 + i);
        }
        const int ng = isize[it].x, gb = ibase[it].x;
        if (tid < kNWK + 1) cp_async<4>(&s_ws[bf][tid], wst + (size_t)it * (kNWK + 1) + tid);
        for (int a = tid; a < ng * 4; a += blockDim.x)
            cp_async<16>((unsigned char*)s_dst[bf] + 16 * a, (const unsigned char*)dest + (size_t)gb * 64 + 16 * a);
    };
    int cur_lg = i0 / nch, slot = 0;
    uint2 va[kStage];   // entry blocks of the warp's current position (prefetched across items)
    bool pre = false;
    if (i0 < i1) issue(i0, 0);
    for (int it = i0; it < i1; it++) {
        const int lg = it / nch, c = it - lg * nch;
        const int bf = (it - i0) & 1;
        cp_async_commit_wait_all();                          // this thread's table copies of item it
        if (tma) mbar_wait(&bars[bf], (uint32_t)(((it - i0) >> 1) & 1));
        CWB_JIT(it * 4 + 0);
        __syncthreads();  // item it's data visible; item it - 1 consumed (buffer bf ^ 1 is free)
        CWB_JIT(it * 4 + 1);
        if (lg != cur_lg) {  // flush the bin sums of the previous learner group
            for (int a = tid; a < NU; a += blockDim.x) {
                Pj[(size_t)slot * NU + a] = U[a];
                U[a] = 0.0;
            }
            slot++;
            cur_lg = lg;
            __syncthreads();
        }
        CWB_JIT(it * 4 + 2);
        if (it + 1 < i1) issue(it + 1, bf ^ 1);
        // this warp's block range in item it + 1, read early: its first blocks are loaded before the
        // end-of-item barrier so that their latency overlaps the wait
        uint32_t nws = 0, nwe = 0;
        if (it + 1 < i1) {
            nws = __ldg(wst + (size_t)(it + 1) * (kNWK + 1) + w);
            nwe = __ldg(wst + (size_t)(it + 1) * (kNWK + 1) + w + 1);
        }
        const double* rs = sm + bf * (kC + kPad);
        const unsigned char* rb = (const unsigned char*)rs;
        if (lg == 0) {  // r^T r of the chunk (I8 / the SSE identity): one writer per chunk, fixed order
            const int len = (int)min((int64_t)kC, n - (int64_t)c * kC);
            double sq = 0.0;
            for (int i = tid; i < len; i += blockDim.x) sq = fma(rs[i], rs[i], sq);
            if (!isfinite(sq)) cwb_dev_fail(status, CWB_ENONFINITE);
            sq = warp_sum(sq);
            if (lane == 0) red[w] = sq;
            __syncthreads();
            if (tid == 0) {
                double t = 0.0;
                for (int u = 0; u < nw; u++) t += red[u];
                rrp[(size_t)q * nch + c] = t;
            }
        }
        // this warp's entry blocks [ws[w], ws[w+1]) (warp-major plan layout): its groups in dealing order,
        // bit 0 of a lane's first entry marks the last block of a group; loads run 4 blocks ahead
        const uint16_t* dss = s_dst[bf];
        const uint32_t bend = s_ws[bf][w + 1];
        uint32_t blk = s_ws[bf][w];
        auto gsn = [&](int jr) { return jr * kNWK + ((jr & 1) ? kNWK - 1 - w : w); };
        int jr = 0, g = gsn(0);
        double a0 = 0.0, a1 = 0.0;
        auto loadS = [&](uint2 (&v)[kStage], uint32_t b) {
#pragma unroll
            for (int u = 0; u < kStage; u++)
                if (b + u < bend) v[u] = __ldg(ent + (size_t)(b + u) * 32 + lane);
        };
        auto procS = [&](const uint2 (&v)[kStage], uint32_t b) {
#pragma unroll
            for (int u = 0; u < kStage; u++) {
                if (b + u >= bend) break;
                if (u & 1) a1 += gather4(rb, v[u]);
                else a0 += gather4(rb, v[u]);
                if (v[u].x & 1u) {  // end of group (warp-uniform): the lane's bin total
                    const uint16_t dst = dss[g * 32 + lane];
                    if (dst != 0xffff) U[dst] += a0 + a1;
                    a0 = a1 = 0.0;
                    g = gsn(++jr);
                }
            }
        };
        uint2 vb[kStage];
        if (!pre) loadS(va, blk);
        for (; blk < bend; blk += 2 * kStage) {
            loadS(vb, blk + kStage);
            procS(va, blk);
            if (blk + kStage >= bend) break;
            loadS(va, blk + 2 * kStage);
            procS(vb, blk + kStage);
        }
        pre = false;
        if (it + 1 < i1) {  // first blocks of item it + 1
#pragma unroll
            for (int u = 0; u < kStage; u++)
                if (nws + u < nwe) va[u] = __ldg(ent + (size_t)(nws + u) * 32 + lane);
            pre = true;
        }
    }
    __syncthreads();
    if (i0 < i1)
        for (int a = tid; a < NU; a += blockDim.x) Pj[(size_t)slot * NU + a] = U[a];
}

// findBestBaselearner tail for B <= 4 columns, one block per learner k, fused with the
// combine of the stream kernel's partials:
//   u_k(l) = sum over CTAs of the partial bin sums            (binMatVec)
//   s = Zb^T u over the design-point window of basis j
//   theta = (G + lambda D)^-1 s with the cached inverse
//   delta = 2 theta^T s - theta^T G theta, SSE = r^T r - delta
// and the last block to finish (atomic ticket) takes argmin SSE over k, lowest k on ties
// (P:L292), for every column.
__global__ void __launch_bounds__(1024, 1) k_fit_narrow(
    const double* __restrict__ P, int K, int ns, int Ks, int nch, int nitems, int N, int nslot, int B, int d, int W,
    const double* __restrict__ ZT, const int32_t* __restrict__ lwin, const double* __restrict__ Ainv,
    const double* __restrict__ G, const double* __restrict__ rrp, double* __restrict__ theta, double* __restrict__ delta,
    unsigned* __restrict__ ticket, int32_t* __restrict__ k_out, double* __restrict__ theta_out,
    double* __restrict__ sse_out) {
    extern __shared__ double u[];  // [ns][B], then this learner's ZT [W][d], A^-1 [d][d], G [d][d]
    __shared__ double S[CWB_MAX_D][4], Th[CWB_MAX_D][4], V[CWB_MAX_D][4];
    __shared__ int s_j[CWB_MAX_SMS + 1], s_slot[CWB_MAX_SMS + 1], s_nj, s_lw[2 * CWB_MAX_D];
    __shared__ bool last;
    __shared__ double hsum[1024];  // slice sums of the split combine (NE * split <= blockDim.x)
    __shared__ long long s_off[CWB_MAX_SMS + 1];  // offset of each contributing CTA's partial (doubles)
    const int k = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
    const int lg = k / Ks, NU = Ks * ns, a0 = (k - lg * Ks) * ns;
    double* zts = u + (((size_t)ns * B + 1) & ~(size_t)1);
    double* ais = zts + (size_t)W * d;
    double* gks = ais + (size_t)d * d;
    // the learner's tables are copied to shared memory (cp.async) while the partials are combined
    for (int a = tid; a < W * d; a += blockDim.x) cp_async<8>(zts + a, ZT + (size_t)k * W * d + a);
    for (int a = tid; a < d * d; a += blockDim.x) {
        cp_async<8>(ais + a, Ainv + (size_t)k * d * d + a);
        cp_async<8>(gks + a, G + (size_t)k * d * d + a);
    }
    if (tid < 2 * d) s_lw[tid] = lwin[(size_t)k * d * 2 + tid];
    // the CTAs whose item range meets [lg nch, (lg+1) nch), and their slot for lg (warp 0, a lane per CTA)
    if (w == 0) {  // (32-bit divisions: nitems * (N + 1) < 2^31 is checked on the host)
        const int it0 = lg * nch, it1 = it0 + nch;
        int jlo = it0 * N / nitems;
        while (jlo > 0 && nitems * jlo / N > it0) jlo--;
        int m = 0;
        for (int base = jlo;; base += 32) {
            const int jj = base + lane;
            int b0 = 0, b1 = 0;
            if (jj < N) {
                b0 = nitems * jj / N;
                b1 = nitems * (jj + 1) / N;
            }
            const bool ov = jj < N && b0 < it1 && b1 > it0 && b0 != b1;
            const bool stop = jj >= N || b0 >= it1;
            const unsigned bal = __ballot_sync(0xffffffffu, ov);
            if (ov && m + __popc(bal & ((1u << lane) - 1u)) < CWB_MAX_SMS + 1) {
                const int pos = m + __popc(bal & ((1u << lane) - 1u));
                s_j[pos] = jj;
                s_slot[pos] = lg - (int)(b0 / nch);
            }
            m = min(CWB_MAX_SMS + 1, m + __popc(bal));
            if (__any_sync(0xffffffffu, stop)) break;
        }
        if (lane == 0) s_nj = m;
    }
    __syncthreads();
    const int nj = s_nj;
    for (int m = tid; m < nj; m += blockDim.x) s_off[m] = ((long long)s_j[m] * nslot + s_slot[m]) * NU;
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");  // k_h1_stream complete: P and rrp visible
    CWB_JIT(k * 4 + 0);
    // u_k(l) for column q: the CTA partials added in CTA order.  When ns * B is below the block size, each
    // element's partials are cut into `split` consecutive slices summed by different threads (sixteen loads in
    // flight each) and the slice sums are added in slice order: one or two L2 round trips instead of nj / 8
    const int NE = ns * B;
    const int split = max(1, min(kFitSplitMax, (int)blockDim.x / NE));
    const int per = (nj + split - 1) / split;
    for (int e2 = tid; e2 < NE * split; e2 += blockDim.x) {
        const int h = e2 / NE, e = e2 - h * NE;
        const int l = e / B, q = e - l * B;
        const double* pq = P + (size_t)q * N * nslot * NU + a0 + l;
        const int m1 = min(nj, (h + 1) * per);
        double v = 0.0;
        int m = h * per;
        for (; m + 16 <= m1; m += 16) {
            long long o[16];
            double t[16];
#pragma unroll
            for (int x = 0; x < 16; x++) o[x] = s_off[m + x];
#pragma unroll
            for (int x = 0; x < 16; x++) t[x] = __ldcg(pq + o[x]);
#pragma unroll
            for (int x = 0; x < 16; x++) v += t[x];
        }
        for (; m < m1; m++) v += pq[s_off[m]];
        if (split == 1) u[e] = v;
        else hsum[e2] = v;
    }
    cp_async_commit_wait_all();
    __syncthreads();
    if (split > 1) {
        for (int e = tid; e < NE; e += blockDim.x) {
            double v = hsum[e];
            for (int h = 1; h < split; h++) v += hsum[h * NE + e];
            u[e] = v;
        }
        __syncthreads();
    }
    // s_j = sum over the design-point window of basis j of Zb[l][j] u(l)   (ZT: window-major basis)
    for (int j = w; j < d; j += nw) {
        const int lb = s_lw[2 * j], le = s_lw[2 * j + 1];
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int x = lane; x < le - lb; x += 32) {
            const double z = zts[(size_t)x * d + j];
#pragma unroll
            for (int q = 0; q < 4; q++)
                if (q < B) acc[q] += z * u[(lb + x) * B + q];
        }
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const double t = warp_sum(acc[q]);
            if (lane == 0 && q < B) S[j][q] = t;
        }
    }
    __syncthreads();
    const int jq = tid / B, qq = tid - jq * B;
    if (tid < d * B) {  // theta = A^-1 s (cached inverse)
        const double* Ai = ais + (size_t)jq * d;
        double t = 0.0;
        for (int jp = 0; jp < d; jp++) t += Ai[jp] * S[jp][qq];
        Th[jq][qq] = t;
        theta[((size_t)k * d + jq) * 4 + qq] = t;
    }
    __syncthreads();
    if (tid < d * B) {  // theta_j (2 s_j - (G theta)_j), G banded (|j - j'| <= 3)
        const double* Gk = gks + (size_t)jq * d;
        double gt = 0.0;
        for (int jp = max(0, jq - (CWB_SPW - 1)); jp <= min(d - 1, jq + CWB_SPW - 1); jp++) gt += Gk[jp] * Th[jp][qq];
        V[jq][qq] = Th[jq][qq] * (2.0 * S[jq][qq] - gt);
    }
    __syncthreads();
    if (tid < B) {
        double v = 0.0;
        for (int j = 0; j < d; j++) v += V[j][tid];
        delta[(size_t)k * 4 + tid] = v;
    }
    CWB_JIT(k * 4 + 1);
    __threadfence();
    __syncthreads();
    if (tid == 0) last = atomicAdd(ticket, 1u) == (unsigned)(K - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (w < B) {  // warp q: argmax delta over k (lowest k on ties), r^T r from the chunk partials
        const int q = w;
        int ks = K;
        double best = 0.0;
        for (int kk = lane; kk < K; kk += 32) {
            const double v = __ldcg(delta + (size_t)kk * 4 + q);
            if (ks == K || v > best) { best = v; ks = kk; }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int ok = __shfl_xor_sync(0xffffffffu, ks, o);
            if (ok < K && (ks == K || ob > best || (ob == best && ok < ks))) { best = ob; ks = ok; }
        }
        double rr = 0.0;
        for (int c = lane; c < nch; c += 32) rr += __ldcg(rrp + (size_t)q * nch + c);
        rr = warp_sum(rr);
        if (lane == 0) {
            if (k_out) k_out[q] = ks;
            if (sse_out) sse_out[q] = rr - best;
        }
        if (theta_out && lane < d) theta_out[(size_t)q * d + lane] = __ldcg(theta + ((size_t)ks * d + lane) * 4 + q);
    }
    if (tid == 0) *ticket = 0u;  // ready for the next call
}

}  // namespace

// ===================================================================== host

void cwb_stream_release(cwb_ctx* c, cudaStream_t s) {
    cwb_stream_plan& p = c->sp;
    cwb_release(p.ent, s); cwb_release(p.gtab, s); cwb_release(p.dest, s); cwb_release(p.isize, s);
    cwb_release(p.ibase, s); cwb_release(p.part, s); cwb_release(p.wst, s);
    p = cwb_stream_plan();
}

// Builds the gather plan (once per pool).  Synchronises the stream once (sizes).
static int stream_plan(cwb_ctx* c, cudaStream_t s) {
    cwb_stream_plan& p = c->sp;
    if (p.ready) return CWB_OK;
    const int K = c->K, ns = c->n_star;
    const int64_t n = c->n;
    if (ns > kUBudget) return CWB_EUNSUPPORTED;  // <= kMaxG groups of 32 tasks per item
    // learner group size Ks: bin sums within the shared-memory budget; among those, the one with the smallest
    // makespan estimate: the CTAs take contiguous item ranges, so the busiest CTA runs ceil(items / SMs) items of
    // Ks learners each plus a fixed per-item cost (chunk staging, barrier; ~3 learners' worth), larger Ks on ties
    const int nch0 = (int)((n + kC - 1) / kC);
    const int nsm = cwb_num_sms();
    int Ks = 1;
    int64_t best = INT64_MAX;
    for (int ks = 1; ks <= std::min(K, kUBudget / ns); ks++) {
        const int64_t items = (int64_t)((K + ks - 1) / ks) * nch0;
        const int64_t cost = ((items + nsm - 1) / nsm) * (ks + 3);
        if (cost <= best) { best = cost; Ks = ks; }
    }
    if ((int64_t)Ks * ns > 0xfffe) return CWB_EUNSUPPORTED;
    const int nch = (int)((n + kC - 1) / kC), nlg = (K + Ks - 1) / Ks, nitems = nlg * nch;
    int NTP = 32;
    while (NTP < Ks * ns) NTP <<= 1;
    if ((size_t)NTP * 8 > 200 * 1024) return CWB_EUNSUPPORTED;
    uint32_t *cnt = nullptr, *cst = nullptr, *tasks = nullptr, *gsteps = nullptr;
    int2 *isize = nullptr, *ibase = nullptr;
    long long* tot = nullptr;
    bool ok = true;
    const size_t nc = (size_t)K * nch * ns;
    ok &= cwb_alloc((void**)&cnt, sizeof(uint32_t) * nc, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&cst, sizeof(uint32_t) * nc, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&tasks, sizeof(uint32_t) * (size_t)nitems * NTP, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&gsteps, sizeof(uint32_t) * (size_t)nitems * (NTP / 32 + 1), s) == cudaSuccess;
    ok &= cwb_alloc((void**)&isize, sizeof(int2) * nitems, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&ibase, sizeof(int2) * nitems, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&tot, sizeof(long long) * 2, s) == cudaSuccess;
    auto cleanup = [&]() {
        cwb_release(cnt, s); cwb_release(cst, s); cwb_release(tasks, s); cwb_release(tot, s); cwb_release(gsteps, s);
    };
    if (!ok) {
        cleanup(); cwb_release(isize, s); cwb_release(ibase, s);
        return cwb_set_error(c, CWB_ENOMEM, "stream plan allocation failed");
    }
    const size_t hsm = sizeof(uint32_t) * ns;
    if (c->idx_bytes == 1)
        k_sp_count<uint8_t><<<dim3(nch, K), 256, hsm, s>>>((const uint8_t*)c->idx, n, ns, nch, cnt);
    else
        k_sp_count<uint16_t><<<dim3(nch, K), 256, hsm, s>>>((const uint16_t*)c->idx, n, ns, nch, cnt);
    k_sp_start<<<(unsigned)(((int64_t)K * ns + 255) / 256), 256, 0, s>>>(cnt, c->off, K, ns, nch, cst);
    const size_t ssm = sizeof(unsigned long long) * NTP;
    cudaFuncSetAttribute(k_sp_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
    k_sp_sort<<<nitems, 512, ssm, s>>>(cnt, K, ns, nch, Ks, NTP, tasks, isize);
    if (c->perm_bytes == 2)
        k_sp_sched<uint16_t, false><<<nitems, 512, 0, s>>>(tasks, cnt, cst, (const uint16_t*)c->perm, n, ns, nch, Ks,
                                                           NTP, isize, ibase, gsteps, nullptr, nullptr, nullptr);
    else
        k_sp_sched<uint32_t, false><<<nitems, 512, 0, s>>>(tasks, cnt, cst, (const uint32_t*)c->perm, n, ns, nch, Ks,
                                                           NTP, isize, ibase, gsteps, nullptr, nullptr, nullptr);
    k_sp_scan<<<1, 1, 0, s>>>(isize, nitems, ibase, tot);
    c->launches += 5;
    long long h_tot[2] = {0, 0};
    cudaMemcpyAsync(h_tot, tot, sizeof(h_tot), cudaMemcpyDeviceToHost, s);
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        cleanup(); cwb_release(isize, s); cwb_release(ibase, s);
        return cwb_set_error(c, CWB_ECUDA, std::string("stream plan: ") + cudaGetErrorString(e));
    }
    const long long ngt = h_tot[0], nbt = h_tot[1];
    if (nbt >= (1ll << 31) / 32 || ngt >= (1ll << 31) / 32) {
        cleanup(); cwb_release(isize, s); cwb_release(ibase, s);
        return CWB_EUNSUPPORTED;
    }
    ok = cwb_alloc((void**)&p.ent, (size_t)std::max(1ll, nbt) * 256, s) == cudaSuccess;
    ok &= cwb_alloc((void**)&p.gtab, sizeof(uint2) * (size_t)std::max(1ll, ngt), s) == cudaSuccess;
    ok &= cwb_alloc((void**)&p.dest, sizeof(uint16_t) * 32 * (size_t)std::max(1ll, ngt), s) == cudaSuccess;
    ok &= cwb_alloc((void**)&p.wst, sizeof(uint32_t) * (kNWK + 1) * (size_t)nitems, s) == cudaSuccess;
    if (!ok) {
        cleanup(); cwb_release(isize, s); cwb_release(ibase, s);
        cwb_stream_release(c, s);
        return cwb_set_error(c, CWB_ENOMEM, "stream plan allocation failed");
    }
    if (c->perm_bytes == 2)
        k_sp_sched<uint16_t, true><<<nitems, 512, 0, s>>>(tasks, cnt, cst, (const uint16_t*)c->perm, n, ns, nch, Ks,
                                                          NTP, isize, ibase, gsteps, (uint16_t*)p.ent, p.gtab, p.dest);
    else
        k_sp_sched<uint32_t, true><<<nitems, 512, 0, s>>>(tasks, cnt, cst, (const uint32_t*)c->perm, n, ns, nch, Ks,
                                                          NTP, isize, ibase, gsteps, (uint16_t*)p.ent, p.gtab, p.dest);
    k_sp_wstart<<<nitems, 32, 0, s>>>(isize, ibase, gsteps, NTP, p.wst);  // kNWK <= 32
    c->launches += 2;
    cleanup();
    p.isize = isize;
    p.ibase = ibase;
    p.Ks = Ks;
    p.nch = nch;
    p.nlg = nlg;
    p.nitems = nitems;
    p.ngroups = ngt;
    p.nblocks = nbt;
    p.ready = true;
    return cwb_check_launch(c, "stream plan kernels");
}

// findBestBaselearner for B <= 4 residual columns R[B][n] (k_out[B], theta_out[B][d], sse_out[B]):
// k_h1_stream + k_fit_narrow.  CWB_EUNSUPPORTED when the plan does not apply (caller falls back).
int cwb_find_best_stream(cwb_ctx* c, const double* R, int32_t B, int32_t* k_out, double* theta_out,
                         double* sse_out, cudaStream_t s) {
    if (c->rows || B < 1 || B > 4 || (size_t)c->n_star * B * sizeof(double) > 96 * 1024 ||
        c->n_star > kUBudget) return CWB_EUNSUPPORTED;
    if ((int64_t)c->K * ((c->n + kC - 1) / kC) * (CWB_MAX_SMS + 1) >= INT32_MAX) return CWB_EUNSUPPORTED;  // item math in int32
    {   // k_fit_narrow stages the bin sums, the window-major basis and two d x d tables in shared memory:
        // larger pools take the other findBest paths
        const size_t fsm0 = sizeof(double) * ((((size_t)c->n_star * B + 1) & ~(size_t)1) + (size_t)c->W * c->d +
                                              2 * (size_t)c->d * c->d);
        cudaFuncAttributes fa;
        int optin = 0, dev = 0;
        if (cudaFuncGetAttributes(&fa, k_fit_narrow) != cudaSuccess || cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) {
            cudaGetLastError();
            return CWB_EUNSUPPORTED;
        }
        if (fsm0 + fa.sharedSizeBytes > (size_t)optin) return CWB_EUNSUPPORTED;
    }
    int rc = stream_plan(c, s);
    if (rc) return rc;
    cwb_stream_plan& p = c->sp;
    const int K = c->K, ns = c->n_star, d = c->d;
    const int N = std::max(1, std::min(p.nitems, cwb_num_sms()));
    // learner groups met by one CTA's item range
    const int per = (p.nitems + N - 1) / N;
    const int nslot = std::min(p.nlg, (per + p.nch - 1) / p.nch + 1);
    const size_t part = (size_t)B * N * nslot * p.Ks * ns, extra = (size_t)4 * p.nch + (size_t)K * (d + 1) * 4 + 1;
    const size_t need = sizeof(double) * (part + extra);
    if (p.part_bytes < need) {
        cwb_release(p.part, s);
        p.part = nullptr;
        p.part_bytes = 0;
        if (cwb_alloc((void**)&p.part, need, s) != cudaSuccess)
            return cwb_set_error(c, CWB_ENOMEM, "stream find_best workspace allocation failed");
        p.part_bytes = need;
        cudaMemsetAsync(p.part + part + extra - 1, 0, sizeof(double), s);  // ticket
    }
    double* rrp = p.part + part;
    double* th = rrp + 4 * p.nch;
    double* de = th + (size_t)K * d * 4;
    unsigned* ticket = (unsigned*)(p.part + part + extra - 1);
    const size_t smem = sizeof(double) * (2 * ((size_t)kC + kPad) + (size_t)p.Ks * ns);
    cudaFuncSetAttribute(k_h1_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_h1_stream<<<dim3(N, B), kStreamT, smem, s>>>(R, c->n, p.nch, p.Ks, ns, p.nitems, nslot, (const uint2*)p.ent,
                                                    p.gtab, p.dest, p.isize, p.ibase, p.wst, p.part, rrp, c->d_status);
    const size_t fsm = sizeof(double) * ((((size_t)ns * B + 1) & ~(size_t)1) + (size_t)c->W * d + 2 * (size_t)d * d);
    CWB_CUDA_TRY(c, cudaFuncSetAttribute(k_fit_narrow, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm));
    static const int no_fit = getenv("CWB_STREAM_NOFIT") ? atoi(getenv("CWB_STREAM_NOFIT")) : 0;
    if (no_fit) {  // timing experiment only (tools/findbest_timing.py): the stream kernel alone, outputs invalid
        c->launches += 1;
        return cwb_check_launch(c, "stream kernel");
    }
    {   // launched as a programmatic dependent of k_h1_stream (prologue overlaps its tail)
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(K);
        lc.blockDim = dim3(1024);
        lc.dynamicSmemBytes = fsm;
        lc.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        CWB_CUDA_TRY(c, cudaLaunchKernelEx(&lc, k_fit_narrow, (const double*)p.part, K, ns, p.Ks, p.nch, p.nitems, N,
                                           nslot, B, d, (int)c->W, (const double*)c->ZT, (const int32_t*)c->lwin,
                                           (const double*)c->Ainv, (const double*)c->G, (const double*)rrp, th, de,
                                           ticket, k_out, theta_out, sse_out));
    }
    c->launches += 2;
    return cwb_check_launch(c, "stream find_best kernels");
}
