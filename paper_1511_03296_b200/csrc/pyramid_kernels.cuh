// pyramid_kernels.cuh — bilateral-space pyramid (Supp. Sec. 2; reading #8).
//
// Level k+1 = unique(⌊V_k / 2⌋) with the frame field kept.  A level-(k+1) vertex lies in the
// coarse cell (⌊by/2⌋, ⌊bx/2⌋); its children are the level-k vertices of the ≤ 2×2 level-k cells
// below it, i.e. two contiguous ranges of the canonical level-k order.  One block per coarse
// cell sorts (halved code, child id) pairs in shared memory, takes unique runs as parents, and a
// decoupled look-back over coarse cells assigns global parent and child-list offsets — the
// level is canonical (ascending key) by construction.
#pragma once
#include "fbs_common.cuh"

namespace fbs {

__device__ __forceinline__ uint32_t halve_code(uint32_t code) {
    const uint32_t l = (code >> 16) & 255u, u = (code >> 8) & 255u, v = code & 255u;
    return ((l >> 1) << 16) | ((u >> 1) << 8) | (v >> 1);
}

// Block-wide exclusive scan of one int per thread (blockDim ≤ 1024).  Returns the exclusive
// prefix; *total receives the sum.  Contains __syncthreads.
__device__ __forceinline__ int block_excl_scan(int x, int* sh /*[33]*/, int* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    __syncthreads();
    if (lane == 31) sh[w] = incl;
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        int s = (lane < nw) ? sh[lane] : 0;
        int si = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, si, o);
            if (lane >= o) si += y;
        }
        if (lane < nw) sh[lane] = si - s;
        if (lane == 31) sh[32] = si;
    }
    __syncthreads();
    *total = sh[32];
    return sh[w] + incl - x;
}

// One block (T threads) per level-(k+1) coarse cell.  One look-back chain carries the packed
// (vertex, child) counts.  Cells with more than kCoarseCap children sort in a global scratch
// slice (rare: dense pixel-noise images at σl = σuv = 1).
__global__ void __launch_bounds__(64) k_pyr_level(
    const uint64_t* __restrict__ keysK, const int* __restrict__ cellOffK, int ncxK, int ncyK,
    int ncxN, int ncyN, int64_t ncellsN, unsigned* __restrict__ tile_counter,
    unsigned long long* __restrict__ stateV, unsigned* __restrict__ bump,
    unsigned long long* __restrict__ scratch, uint64_t* __restrict__ keysN,
    int* __restrict__ parentK, int* __restrict__ childStartN, int* __restrict__ childListN,
    int* __restrict__ cellOffN) {
    extern __shared__ unsigned long long sk_smem[];  // [kCoarseCap]
    __shared__ unsigned s_tile;
    __shared__ int s_scan[33];
    __shared__ unsigned s_scr;
    __shared__ unsigned long long s_vexcl;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const int64_t C = s_tile;
    const int T = blockDim.x;

    int f = 0, CY = 0, CX = 0, n0 = 0, n1 = 0, s0 = 0, s1 = 0;
    {
        const int64_t per = (int64_t)ncxN * ncyN;
        f = (int)(C / per);
        const int64_t r = C - (int64_t)f * per;
        CY = (int)(r / ncxN);
        CX = (int)(r - (int64_t)CY * ncxN);
        const int cx0 = 2 * CX, cx1 = min(2 * CX + 1, ncxK - 1);
        for (int a = 0; a < 2; ++a) {
            const int cy = 2 * CY + a;
            if (cy >= ncyK) continue;
            const int64_t ck = ((int64_t)f * ncyK + cy) * ncxK + cx0;
            const int st = cellOffK[ck], en = cellOffK[ck + (cx1 - cx0) + 1];
            if (a == 0) { s0 = st; n0 = en - st; } else { s1 = st; n1 = en - st; }
        }
    }
    const int nch = n0 + n1;
    int P = 1;
    while (P < nch) P <<= 1;
    // oversize cells sort in a global scratch slice taken from a bump allocator (its position
    // does not affect the result); Σ P < 2·M bounds the scratch
    if (threadIdx.x == 0) s_scr = (nch > kCoarseCap) ? atomicAdd(bump, (unsigned)P) : 0u;
    __syncthreads();
    unsigned long long* sk = (nch <= kCoarseCap) ? sk_smem : scratch + s_scr;
    for (int i = threadIdx.x; i < P; i += T) {
        unsigned long long key = ~0ull;
        if (i < nch) {
            const int gch = (i < n0) ? s0 + i : s1 + (i - n0);
            key = ((unsigned long long)halve_code((uint32_t)(keysK[gch] & 0xffffffu)) << 32) | (unsigned)gch;
        }
        sk[i] = key;
    }
    __syncthreads();
    // bitonic sort of P (power of two) keys
    for (int k = 2; k <= P; k <<= 1) {
        for (int s = k >> 1; s > 0; s >>= 1) {
            for (int i = threadIdx.x; i < P; i += T) {
                const int j = i ^ s;
                if (j > i) {
                    const bool asc = (i & k) == 0;
                    const unsigned long long a = sk[i], b = sk[j];
                    if ((a > b) == asc) { sk[i] = b; sk[j] = a; }
                }
            }
            __syncthreads();
        }
    }
    // heads and ranks: thread t owns elements [t*E, t*E + E)
    const int E = (nch + T - 1) / T;
    const int i0 = threadIdx.x * E;
    int myHeads = 0;
    for (int e = 0; e < E; ++e) {
        const int i = i0 + e;
        if (i < nch && (i == 0 || (sk[i] >> 32) != (sk[i - 1] >> 32))) ++myHeads;
    }
    int U;
    const int before = block_excl_scan(myHeads, s_scan, &U);
    if (threadIdx.x < 32) {
        const unsigned long long ex = lookback_warp(stateV, (unsigned)C, lb_pack((unsigned)U, (unsigned)nch));
        if (threadIdx.x == 0) s_vexcl = ex;
    }
    __syncthreads();
    const int vOff = (int)lb_first(s_vexcl), cOff = (int)lb_second(s_vexcl);
    const uint64_t khi = ((uint64_t)f << 56) | ((uint64_t)CY << 40) | ((uint64_t)CX << 24);
    int r = before - 1;
    for (int e = 0; e < E; ++e) {
        const int i = i0 + e;
        if (i >= nch) break;
        const bool head = (i == 0 || (sk[i] >> 32) != (sk[i - 1] >> 32));
        if (head) ++r;
        const int gch = (int)(sk[i] & 0xffffffffull);
        parentK[gch] = vOff + r;
        childListN[cOff + i] = gch;
        if (head) {
            keysN[vOff + r] = khi | (sk[i] >> 32);
            childStartN[vOff + r] = cOff + i;
        }
    }
    if (threadIdx.x == 0) {
        cellOffN[C] = vOff;
        if (C == ncellsN - 1) {
            cellOffN[ncellsN] = vOff + U;
            childStartN[vOff + U] = cOff + nch;
        }
    }
}

// P(1) at level k+1 from level k (segment sums over the child lists; integers, exact).
__global__ void k_lift_count(const int* __restrict__ countK, const int* __restrict__ childStart,
                             const int* __restrict__ childList, int Mn, int* __restrict__ countN) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < Mn; p += gridDim.x * blockDim.x) {
        int s = 0;
        for (int j = childStart[p]; j < childStart[p + 1]; ++j) s += countK ? countK[childList[j]] : 1;
        countN[p] = s;
    }
}

// frame offsets of a level from its cell offsets: frameOff[f] = cellOff[f * ncx * ncy]
__global__ void k_frame_offsets(const int* __restrict__ cellOff, int F, int64_t cellsPerFrame,
                                int* __restrict__ frameOff) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f <= F) frameOff[f] = cellOff[(int64_t)f * cellsPerFrame];
}

}  // namespace fbs
