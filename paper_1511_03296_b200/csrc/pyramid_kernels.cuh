// pyramid_kernels.cuh — bilateral-space pyramid (Supp. Sec. 2; reading #8).
//
// Level k+1 = unique(⌊V_k / 2⌋) with the frame field kept.  A level-(k+1) vertex lies in the
// coarse cell (⌊by/2⌋, ⌊bx/2⌋); its children are the level-k vertices of the ≤ 2×2 level-k cells
// below it, i.e. two contiguous ranges of the canonical level-k order.  Per level: one block per
// coarse cell sorts (halved code, child id) pairs and takes unique runs as parents (k_pyr_sort),
// an exclusive scan of the parent counts gives the global parent offsets (k_scan_excl), and
// k_pyr_write assigns the canonical parent ids — the level is canonical (ascending key) by
// construction.
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

// Coarse cell C = (f, CY, CX) of level k+1 covers the level-k cells (2CY..2CY+1, 2CX..2CX+1): its
// children are two contiguous ranges [s0, s0+n0) (row 2CY) and [s1, s1+n1) (row 2CY+1), and its
// child-list offset has a closed form — the children of all earlier coarse cells are the level-k
// vertices of earlier level-k rows plus those left of column 2CX in rows 2CY and 2CY+1.
struct CoarseCell {
    int f, CY, CX, s0, n0, s1, n1, cOff;
};
__device__ __forceinline__ CoarseCell coarse_cell(int64_t C, const int* __restrict__ cellOffK, int ncxK, int ncyK,
                                                  int ncxN, int ncyN) {
    CoarseCell cc{};
    const unsigned per = (unsigned)ncxN * (unsigned)ncyN, cu = (unsigned)C;  // 32-bit: cell counts < 2^31
    cc.f = (int)(cu / per);
    const unsigned r = cu - (unsigned)cc.f * per;
    cc.CY = (int)(r / (unsigned)ncxN);
    cc.CX = (int)(r - (unsigned)cc.CY * (unsigned)ncxN);
    const int cx0 = 2 * cc.CX, cx1 = min(2 * cc.CX + 1, ncxK - 1);
    const int64_t ck0 = ((int64_t)cc.f * ncyK + 2 * cc.CY) * ncxK;
    cc.s0 = cellOffK[ck0 + cx0];
    cc.n0 = cellOffK[ck0 + cx1 + 1] - cc.s0;
    cc.cOff = cc.s0;
    if (2 * cc.CY + 1 < ncyK) {
        const int64_t ck1 = ck0 + ncxK;
        cc.s1 = cellOffK[ck1 + cx0];
        cc.n1 = cellOffK[ck1 + cx1 + 1] - cc.s1;
        cc.cOff += cc.s1 - cellOffK[ck1];
    }
    return cc;
}

// Bitonic sort of 32·E keys held in a warp's registers, blocked layout (lane l holds elements
// l·E .. l·E + E − 1): strides ≥ E exchange across lanes with shuffles, smaller ones inside a lane.
template <int E, typename KeyT = unsigned long long>
__device__ __forceinline__ void warp_bitonic(KeyT (&key)[E]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int kk = 2; kk <= 32 * E; kk <<= 1) {
#pragma unroll
        for (int sd = kk >> 1; sd > 0; sd >>= 1) {
            if (sd >= E) {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int i = lane * E + e;
                    const KeyT o = __shfl_xor_sync(0xffffffffu, key[e], sd / E);
                    const bool keepMin = ((i & sd) == 0) == ((i & kk) == 0);
                    key[e] = keepMin ? (key[e] < o ? key[e] : o) : (key[e] < o ? o : key[e]);
                }
            } else {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int pe = e ^ sd;
                    if (pe > e) {
                        const bool asc = ((lane * E + e) & kk) == 0;
                        const KeyT a = key[e], b = key[pe];
                        const bool sw = (a > b) == asc;
                        key[e] = sw ? b : a;
                        key[pe] = sw ? a : b;
                    }
                }
            }
        }
    }
}

__device__ __forceinline__ unsigned long long child_key(const uint64_t* __restrict__ keysK, const CoarseCell& cc,
                                                        int i) {
    const int gch = (i < cc.n0) ? cc.s0 + i : cc.s1 + (i - cc.n0);
    return ((unsigned long long)halve_code((uint32_t)(keysK[gch] & 0xffffffu)) << 32) | (unsigned)gch;
}

// ≤ 32·E ≤ 128 children sorted in registers as 32-bit keys (halved code ‖ 7-bit child index in
// the cell: 64-bit compares ran the math pipe at its limit); the child index orders exactly like the
// global child id (row 2CY's range precedes row 2CY+1's), so the order equals that of
// (code, child id).  Heads (first child of each parent code) → parent ranks.
template <int E>
__device__ __forceinline__ int pyr_sort_regs(const uint64_t* __restrict__ keysK, const CoarseCell& cc, int nch,
                                             int* __restrict__ childListN, int* __restrict__ rankS) {
    static_assert(32 * E <= 128, "7-bit child index");
    const int lane = threadIdx.x & 31;
    uint32_t key[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = lane * E + e;
        uint32_t k = 0xffffffffu;
        if (i < nch) {
            const int gch = (i < cc.n0) ? cc.s0 + i : cc.s1 + (i - cc.n0);
            k = (halve_code((uint32_t)(keysK[gch] & 0xffffffu)) << 7) | (uint32_t)i;
        }
        key[e] = k;
    }
    warp_bitonic<E, uint32_t>(key);
    const uint32_t hiPrevLane = __shfl_up_sync(0xffffffffu, key[E - 1] >> 7, 1);
    int heads = 0;
    unsigned hm = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = lane * E + e;
        const uint32_t prev = (e == 0) ? hiPrevLane : (key[e - 1] >> 7);
        const bool head = i < nch && (i == 0 || (key[e] >> 7) != prev);
        hm |= (unsigned)head << e;
        heads += head;
    }
    int incl = heads;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    int r = incl - heads - 1;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = lane * E + e;
        if (i < nch) {
            r += (hm >> e) & 1u;
            const int li = (int)(key[e] & 127u);
            childListN[cc.cOff + i] = (li < cc.n0) ? cc.s0 + li : cc.s1 + (li - cc.n0);
            rankS[cc.cOff + i] = r;
        }
    }
    return __shfl_sync(0xffffffffu, incl, 31);
}


// Pass 1: one warp per coarse cell sorts its (halved code, child id) pairs — in registers (32-bit keys) for
// ≤ 128 children (the typical level-1 cell), else in a global scratch
// slice from a bump allocator — writes the children grouped by parent in canonical order to the
// child list, each sorted position's parent rank (rankS) and the cell's parent count.  Warps are
// independent (no inter-block chain, no shared memory).
__global__ void __launch_bounds__(256) k_pyr_sort(const uint64_t* __restrict__ keysK, const int* __restrict__ cellOffK,
                                                  int ncxK, int ncyK, int ncxN, int ncyN, int64_t ncellsN,
                                                  unsigned* __restrict__ bump, unsigned long long* __restrict__ scratch,
                                                  int* __restrict__ childListN, int* __restrict__ rankS,
                                                  int* __restrict__ cnt) {
    pdl_entry();
    const int lane = threadIdx.x & 31;
    for (int64_t C = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; C < ncellsN;
         C += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const CoarseCell cc = coarse_cell(C, cellOffK, ncxK, ncyK, ncxN, ncyN);
        const int nch = cc.n0 + cc.n1;
        int U;
        if (nch <= 32) U = pyr_sort_regs<1>(keysK, cc, nch, childListN, rankS);
        else if (nch <= 64) U = pyr_sort_regs<2>(keysK, cc, nch, childListN, rankS);
        else if (nch <= 128) U = pyr_sort_regs<4>(keysK, cc, nch, childListN, rankS);
        else {
            int P = 1;
            while (P < nch) P <<= 1;
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(bump, (unsigned)P);
            unsigned long long* sk = scratch + __shfl_sync(0xffffffffu, base, 0);
            for (int i = lane; i < P; i += 32) sk[i] = (i < nch) ? child_key(keysK, cc, i) : ~0ull;
            __syncwarp();
            for (int kk = 2; kk <= P; kk <<= 1) {
                for (int sd = kk >> 1; sd > 0; sd >>= 1) {
                    for (int i = lane; i < P; i += 32) {
                        const int j = i ^ sd;
                        if (j > i) {
                            const unsigned long long a = sk[i], b = sk[j];
                            if ((a > b) == ((i & kk) == 0)) {
                                sk[i] = b;
                                sk[j] = a;
                            }
                        }
                    }
                    __syncwarp();
                }
            }
            int r = -1;
            for (int i0 = 0; i0 < nch; i0 += 32) {
                const int i = i0 + lane;
                const bool head = i < nch && (i == 0 || (sk[i] >> 32) != (sk[i - 1] >> 32));
                const unsigned hb = __ballot_sync(0xffffffffu, head);
                if (i < nch) {
                    childListN[cc.cOff + i] = (int)(sk[i] & 0xffffffffull);
                    rankS[cc.cOff + i] = r + __popc(hb & ((2u << lane) - 1u));
                }
                r += __popc(hb);
            }
            U = r + 1;
        }
        if (lane == 0) cnt[C] = U;
    }
}

// Pass 3 (after the exclusive scan of the parent counts → cellOffN): parents get their canonical
// ids vOff + rank: parent map, parent keys and child-list starts, and (summed over each parent's
// children in child order, integers) P(1) = level-0 descendants (countK = nullptr: level 0, one
// each) and the level-1 descendant counts cnt1 (cnt1K = nullptr: the children are level-1
// vertices, one each; cnt1N = nullptr: not needed at level 1).  One warp per coarse cell, 32
// sorted children per round: the per-parent sums are warp segmented scans over the rank runs,
// carried across rounds.
__global__ void __launch_bounds__(256) k_pyr_write(const uint64_t* __restrict__ keysK, const int* __restrict__ cellOffK,
                                                   int ncxK, int ncyK, int ncxN, int ncyN, int64_t ncellsN,
                                                   const int* __restrict__ cellOffN, const int* __restrict__ childListN,
                                                   const int* __restrict__ rankS, uint64_t* __restrict__ keysN,
                                                   int* __restrict__ parentK, int* __restrict__ childStartN,
                                                   const int* __restrict__ countK, int* __restrict__ countN,
                                                   const int* __restrict__ cnt1K, int* __restrict__ cnt1N) {
    pdl_entry();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t C = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; C < ncellsN;
         C += (int64_t)gridDim.x * (blockDim.x >> 5)) {
        const CoarseCell cc = coarse_cell(C, cellOffK, ncxK, ncyK, ncxN, ncyN);
        const int nch = cc.n0 + cc.n1;
        const int vOff = cellOffN[C];
        const uint64_t khi = ((uint64_t)cc.f << 56) | ((uint64_t)cc.CY << 40) | ((uint64_t)cc.CX << 24);
        int carryR = -1, carry0 = 0, carry1 = 0;  // the run still open at the end of the last round
        for (int base = 0; base < nch; base += 32) {
            const int i = base + lane;
            const bool in = i < nch;
            int gch = 0, r = -1 - lane, v0 = 0, v1 = 0;  // distinct dummy ranks past the end
            if (in) {
                gch = childListN[cc.cOff + i];
                r = rankS[cc.cOff + i];
                v0 = countK ? countK[gch] : 1;
                if (cnt1N) v1 = cnt1K ? cnt1K[gch] : 1;
                parentK[gch] = vOff + r;
            }
            const int rPrev = __shfl_up_sync(0xffffffffu, r, 1);
            const bool runHead = (lane == 0) || (r != rPrev);  // first of its run in this round
            if (in && (lane == 0 ? r != carryR : r != rPrev)) {  // first child of parent r
                keysN[vOff + r] = khi | (uint64_t)halve_code((uint32_t)(keysK[gch] & 0xffffffu));
                childStartN[vOff + r] = cc.cOff + i;
            }
            if (lane == 0 && carryR >= 0 && r != carryR) {  // the open run ended at the round boundary
                countN[vOff + carryR] = carry0;
                if (cnt1N) cnt1N[vOff + carryR] = carry1;
            }
            const unsigned hm = __ballot_sync(0xffffffffu, runHead) & ((lane == 31) ? 0xffffffffu : ((2u << lane) - 1u));
            const int sst = 31 - __clz(hm);
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {  // segmented inclusive scans (integers: exact)
                const int t0 = __shfl_up_sync(0xffffffffu, v0, d);
                const int t1 = __shfl_up_sync(0xffffffffu, v1, d);
                if (lane - d >= sst) {
                    v0 += t0;
                    v1 += t1;
                }
            }
            if (sst == 0 && r == carryR) {
                v0 += carry0;
                v1 += carry1;
            }
            const int rNext = __shfl_down_sync(0xffffffffu, r, 1);
            if (in && (i == nch - 1 || (lane < 31 && rNext != r))) {  // run ends inside this round
                countN[vOff + r] = v0;
                if (cnt1N) cnt1N[vOff + r] = v1;
            }
            carryR = __shfl_sync(0xffffffffu, r, 31);
            carry0 = __shfl_sync(0xffffffffu, v0, 31);
            carry1 = __shfl_sync(0xffffffffu, v1, 31);
            if (base + 32 >= nch) carryR = -1;  // the last round closed every run
        }
        if (C == ncellsN - 1 && lane == 0) childStartN[cellOffN[ncellsN]] = cc.cOff + nch;
    }
}

}  // namespace fbs
