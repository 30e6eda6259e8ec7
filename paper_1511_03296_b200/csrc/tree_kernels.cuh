// tree_kernels.cuh — the hierarchical preconditioner and initialisation in tree order
// (Eq. hier_precond, hier init PAPER.md:287-293, pyramid PAPER.md:745-766).
//
// P lifts y through the pyramid, Pᵀ projects back (:763), and both hierarchical
// operators are  out = Pᵀ(mult ∘ P(in))  with per-level multipliers (reading #8: level 0 = y).
// TREE ORDER.  At grid build the level-1 vertices (and the level-0 vertices) are numbered in
// depth-first order of the pyramid (siblings in canonical child order), so the level-1
// descendants of ANY coarse vertex a (level ≥ 2) are one contiguous range rng(a) of the
// tree-ordered level-1 vector.  Hence, per (frame, channel):
//   (P y)_a = Π(end_a) − Π(start_a − 1),   Π = fp64 inclusive prefix of the tree-ordered (P y)_1,
// and the projection of the levels ≥ 2 onto a level-2 vertex a is one ancestor-chain walk
//   acc2_a = Σ_{k≥2} mult_k(anc_k(a))·(P y)_{anc_k(a)},
// handed to its children (one contiguous tree range): acc1_i = mult_1(i)·(P y)_1,i + acc2_{parent(i)}.
// No level-by-level synchronisation remains: one lift+scan pass over level 1, one pass over
// level 2 for all coarse values, one pass over level 0.  Every sum has a fixed order (child
// order, fixed scan trees), so results are bitwise reproducible.
//
// PCG (Alg. 2) uses M⁻¹ = mask∘Pᵀ(μ∘P(mask∘·)), so ρ = rᵀM⁻¹r = Σ_k Σ_a μ_k,a (P w)²_a with
// w = mask∘r: ρ is complete after the lift, and the projection is fused with d = s + βd.
#pragma once
#include "fbs_common.cuh"
#include "solve_kernels.cuh"

namespace fbs {

#ifndef FBS_L0B
#define FBS_L0B 4
#endif
#ifndef FBS_UPB
#define FBS_UPB 4
#endif
constexpr int kL0B = FBS_L0B;  // vertices per round of k_tree_level0 (loads in flight per thread)
constexpr int kUpB = FBS_UPB;  // vertices per round of k_hier_level0

enum { HIER_PCG = 0, HIER_PDA = 1, HIER_INIT = 2, HIER_PLAIN = 3 };
enum { HSRC_UPDATE = 0, HSRC_RESID = 1, HSRC_RESID0 = 2 };

// INIT multiplier z_w(k)/P(1)_k; 0 above the frame's top level (reading #8).
// h.zw[k] = α^−(β+k) of the current use (host-computed).
__device__ __forceinline__ float init_mult1(const HierArgs& h, int k, int fl, int count) {
    return (k < fl) ? (float)(h.zw[k] / (double)count) : 0.f;
}

// μ_k = z_w(k) P(1) / den (Eq. hier_precond)
__device__ __forceinline__ float zw_count(const HierArgs& h, int k, int count, double den) {
    return (float)(h.zw[k] * (double)count / den);
}

// ================================================================ grid build: tree order
// start positions of the top vertex of each frame: its frame's first level-0 / level-1 positions
// (top ≥ 2: also its level-1 range)
__global__ void k_tree_top(const int* __restrict__ lvFrameOff, int F, int top, int2* __restrict__ startTop,
                           int2* __restrict__ rngTop, const int* __restrict__ cnt1Top) {
    pdl_entry();
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < F; f += gridDim.x * blockDim.x) {
        const int F1 = F + 1;
        const int a = lvFrameOff[top * F1 + f];
        if (a < lvFrameOff[top * F1 + f + 1]) {
            startTop[a] = make_int2(lvFrameOff[f], lvFrameOff[F1 + f]);
            if (rngTop) rngTop[a] = make_int2(lvFrameOff[F1 + f], cnt1Top[a]);
        }
    }
}

// Levels of each frame: the first level with a single vertex (reading #8: halving until one
// vertex per frame); a frame with ≤ 1 vertex has 1 level.  lvFrameOff [L][F + 1].
__global__ void k_frame_levels(const int* __restrict__ lvFrameOff, int F, int L, int* __restrict__ frameLevels) {
    pdl_entry();
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= F) return;
    const int F1 = F + 1;
    int Lf = 1;
    if (lvFrameOff[f + 1] - lvFrameOff[f] > 1) {
        Lf = L;
        for (int k = 1; k < L; ++k)
            if (lvFrameOff[k * F1 + f + 1] - lvFrameOff[k * F1 + f] == 1) {
                Lf = k + 1;
                break;
            }
    }
    frameLevels[f] = Lf;
}

// Prefix-scan tiles of the tree-ordered level 1: kScanTile positions, never crossing a frame.
// Block f: tileFrameOff[f] (= Σ_{g<f} ⌈M1_g / kScanTile⌉; block 0 also writes [F]) and the ranges
// and frame of frame f's tiles.  lv1 = level-1 frame offsets [F + 1].
__global__ void k_scan_tiles(const int* __restrict__ lv1, int F, int* __restrict__ tileFrameOff,
                             int2* __restrict__ tileRange, int* __restrict__ tileFrame) {
    pdl_entry();
    __shared__ int sh[33];
    const int f = blockIdx.x;
    int part = 0;  // tiles of frames g < f (+ block 0: all frames for tileFrameOff[F])
    const int lim = (f == 0) ? F : f;
    for (int g = threadIdx.x; g < lim; g += blockDim.x) part += (lv1[g + 1] - lv1[g] + kScanTile - 1) / kScanTile;
    int tot;
    (void)block_excl_scan(part, sh, &tot);
    int before = 0;
    if (f == 0) {
        if (threadIdx.x == 0) {
            tileFrameOff[0] = 0;
            tileFrameOff[F] = tot;
        }
    } else {
        before = tot;
        if (threadIdx.x == 0) tileFrameOff[f] = before;
    }
    const int b0 = lv1[f], b1 = lv1[f + 1];
    const int nt = (b1 - b0 + kScanTile - 1) / kScanTile;
    for (int t = threadIdx.x; t < nt; t += blockDim.x) {
        const int a0 = b0 + t * kScanTile;
        tileRange[before + t] = make_int2(a0, min(a0 + kScanTile, b1));
        tileFrame[before + t] = f;
    }
}

// level k → k−1: each level-k vertex hands consecutive sub-ranges (in canonical child order) of
// its level-0 / level-1 tree ranges to its children.  cnt0 = P(1) of level k−1, cnt1 = level-1
// descendants of level k−1 (k−1 ≥ 2).  k−1 = 1: writes tord1, csT; k−1 = 0: writes tord0;
// k−1 ≥ 2: writes rng = (level-1 start, level-1 count).
__global__ void k_tree_down(int km1, const int* __restrict__ childStart, const int* __restrict__ childList,
                            const int* __restrict__ MkDev, const int2* __restrict__ startK, const int* __restrict__ cnt0,
                            const int* __restrict__ cnt1, int2* __restrict__ startKm1, int2* __restrict__ rngKm1,
                            int* __restrict__ tord0, int* __restrict__ tord1, int* __restrict__ csT) {
    pdl_entry();
    const int Mk = *MkDev;  // level-k vertex count (device)
    for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < Mk; a += gridDim.x * blockDim.x) {
        int2 r = startK[a];
        for (int q = childStart[a]; q < childStart[a + 1]; ++q) {
            const int c = childList[q];
            if (km1 == 0) {
                tord0[r.x] = c;
                r.x += 1;
            } else {
                startKm1[c] = r;
                if (km1 == 1) {
                    tord1[r.y] = c;
                    csT[r.y] = r.x;
                    r.y += 1;
                } else {
                    rngKm1[c] = make_int2(r.y, cnt1[c]);
                    r.y += cnt1[c];
                }
                r.x += cnt0[c];
            }
        }
    }
}

// parent0T[v] = tree position of v's level-1 parent; csT[M1] = M0.
__global__ void k_tree_finish(const int* __restrict__ parent0, const int2* __restrict__ start1,
                              const int* __restrict__ M0Dev, const int* __restrict__ M1Dev, int* __restrict__ parent0T,
                              int* __restrict__ csT) {
    pdl_entry();
    const int64_t M0 = *M0Dev, M1 = *M1Dev;  // level-0 / level-1 vertex counts (device)
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t v = t0; v < M0; v += stride) parent0T[v] = start1[parent0[v]].y;
    if (t0 == 0) csT[M1] = (int)M0;
}

// Ancestor tables of the level-2 vertices (k = 3..top, row k−3): ancId = the level-k ancestor,
// ancRng = its level-1 range.  The PCG coarse pass then reads a whole ancestor chain in one
// coalesced round instead of top−2 dependent (and, after each iteration's streams, DRAM) loads.
__global__ void k_tree_anc(HierArgs h, const int* __restrict__ M2Dev, int* __restrict__ ancId,
                           int2* __restrict__ ancRng) {
    pdl_entry();
    const int top = h.L - 1;
    const int64_t M2 = h.M2;     // row stride (level-2 capacity)
    const int64_t n2 = *M2Dev;   // level-2 vertex count (device)
    for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < n2; a += (int64_t)gridDim.x * blockDim.x) {
        int an = (int)a;
        for (int k = 3; k <= top; ++k) {
            an = h.lv[k - 1].parent[an];
            ancId[(size_t)(k - 3) * M2 + a] = an;
            ancRng[(size_t)(k - 3) * M2 + a] = h.lv[k].rng[an];
        }
    }
}

// per use: ancMult[k−3][a] = the multiplier of the level-k ancestor of level-2 vertex a:
// μ_k (PCG/PLAIN) or z_w(k)/P(1)_k (INIT).  Blocks per frame (h.bpf2).
template <int MODE>
__global__ void k_tree_anc_mult(HierArgs h, const int* __restrict__ ancId, float* __restrict__ ancMult) {
    pdl_entry();
    const int f = blockIdx.x / h.bpf2, j = blockIdx.x % h.bpf2;
    const int F1 = h.F + 1;
    const int top = h.L - 1;
    const int fl = h.frameLevels[f];
    const int64_t M2 = h.M2;  // row stride (level-2 capacity)
    const int a0 = h.lvFrameOff[2 * F1 + f], a1 = h.lvFrameOff[2 * F1 + f + 1];
    for (int a = a0 + j * blockDim.x + threadIdx.x; a < a1; a += h.bpf2 * blockDim.x)
        for (int k = 3; k <= top; ++k) {
            const int id = ancId[(size_t)(k - 3) * M2 + a];
            ancMult[(size_t)(k - 3) * M2 + a] =
                (MODE == HIER_INIT) ? init_mult1(h, k, fl, h.lv[k].count[id]) : h.lv[k].mu[id];
        }
}

// ================================================================ level 0 → PCG input
// w = mask∘r with r from the PCG update r −= αq (Alg. 2 line 9), the initial residual r = b − A x
// (line 2), or r = b (x = 0, backward); partials ρ_0 = Σ μ0 w² and ‖r‖².  The x update x += αd
// (line 8) is done by the next direction pass (k_tree_level0, which streams d anyway), except in
// the FINISH_LAST kernel of the final FIXED-mode iteration.  FINISH_LAST: the
// final FIXED-mode iteration needs no new direction: its last block per frame records ‖r‖² and
// the iteration count and retires the channel.
template <int SRC, bool FINISH_LAST, bool KS = false>
__global__ void __launch_bounds__(256) k_hier_level0(VecArgs a, float* __restrict__ w0) {
    pdl_entry();
    __shared__ double shd[32];
    __shared__ int sflag;
    int f, j, kB, kE, ci;  // frame, part, channels [kB, kE), last-block counter index
    if constexpr (KS) {    // channel split (K > 1): one (frame, channel) per block group
        const int g = blockIdx.x / a.BPF;
        j = blockIdx.x - g * a.BPF;
        f = g / a.K;
        kB = g - f * a.K;
        kE = kB + 1;
        ci = g;
    } else {
        f = blockIdx.x / a.BPF;
        j = blockIdx.x % a.BPF;
        kB = 0;
        kE = a.K;
        ci = f;
    }
    const int v0 = a.frameOff[f], v1 = a.frameOff[f + 1];
    const int stride = a.BPF * blockDim.x;
    for (int k = kB; k < kE; ++k) {
        const int fk = f * a.K + k;
        double rho = 0.0, rr = 0.0;
        if (SRC != HSRC_UPDATE || a.sc_.active[fk]) {
            const size_t off = (size_t)k * a.M;
            const float al = (SRC == HSRC_UPDATE) ? (float)a.sc_.alpha[fk] : 0.f;
            // the initial residual applies A per vertex (gathers): one vertex per round keeps its
            // register count, and with it the occupancy, of a gather kernel
            constexpr int UB = (SRC == HSRC_RESID) ? 1 : kUpB;
            for (int vb = v0 + j * blockDim.x + threadIdx.x; vb < v1; vb += UB * stride) {
                float rv[UB], mv[UB];
                if (SRC == HSRC_UPDATE) {
                    float xv[UB], dv[UB], qv[UB];
#pragma unroll
                    for (int u = 0; u < UB; ++u) {
                        const int v = vb + u * stride;
                        if (v < v1) {
                            if (FINISH_LAST) {
                                xv[u] = a.x[off + v];
                                dv[u] = a.dn[(size_t)k * a.ldn + v].x;
                            }
                            rv[u] = a.r[off + v];
                            qv[u] = a.q[off + v];
                            mv[u] = a.mu0[v];
                        }
                    }
#pragma unroll
                    for (int u = 0; u < UB; ++u) {
                        const int v = vb + u * stride;
                        if (v < v1) {
                            if (FINISH_LAST) a.x[off + v] = xv[u] + al * dv[u];
                            rv[u] -= al * qv[u];
                        }
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < UB; ++u) {
                        const int v = vb + u * stride;
                        if (v < v1) {
                            rv[u] = a.b[off + v];
                            if (SRC == HSRC_RESID) rv[u] -= apply_A_row(a.x + off, a.n, v, a.nbr[v], a.lam, a.sc[v]);
                            mv[u] = a.mu0[v];
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < UB; ++u) {
                    const int v = vb + u * stride;
                    if (v >= v1) continue;
                    a.r[off + v] = rv[u];
                    const float w = (mv[u] > 0.f) ? rv[u] : 0.f;
                    if (!FINISH_LAST && w0) w0[off + v] = w;
                    rr += (double)rv[u] * (double)rv[u];
                    rho += (double)mv[u] * (double)w * (double)w;
                }
            }
        }
        write_partials(a, f, j, k, rho, rr, shd);
    }
    if (FINISH_LAST && last_block_t0(a.counters + ci, a.BPF, &sflag)) {
        for (int k = kB; k < kE; ++k) {
            const int fk = f * a.K + k;
            if (!a.sc_.active[fk]) continue;
            double RR = 0.0;
            for (int jj = threadIdx.x; jj < a.BPF; jj += blockDim.x)
                RR += __ldcg(a.partial + ((size_t)f * a.BPF + jj) * 2 * a.K + 2 * k + 1);
            RR = block_sum(RR, shd);
            if (threadIdx.x == 0) {
                a.sc_.rr[fk] = RR;
                a.sc_.iters[fk] += 1;
                a.sc_.active[fk] = 0;
                atomicSub(a.sc_.n_active, 1);
            }
        }
    }
}

// ================================================================ lift 0 → 1 and the prefix scan
// Work item = (scan tile of kScanTile consecutive tree positions of one frame, channel); blocks
// walk the items of their frame group (tile range read on the device).  Warp w lifts positions
// [32w, 32w + 32): the children of its 32 level-1 vertices are one contiguous range of level-0
// tree positions, staged (coalesced index load + gather) in shared memory and summed by each lane
// over its own children in canonical child order.  Then a fixed-tree fp64 block scan gives the
// within-tile inclusive prefix and the tile total.  The block that completes the last tile of a
// (frame, channel) (per-frame counter) scans that frame's tile totals in a fixed order into the
// exclusive tile bases the coarse pass reads (tileBase): deterministic, no shared-memory limit on
// the frame size, and the scan is done once instead of once per coarse block.
constexpr int kLiftStage = 256;

__device__ __forceinline__ double block_incl_scan_d(double x, double* sh /*[32]*/, double* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    __syncthreads();
    if (lane == 31) sh[w] = incl;
    __syncthreads();
    if (w == 0) {
        double s = (lane < nw) ? sh[lane] : 0.0;
        double si = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, si, o);
            if (lane >= o) si += y;
        }
        if (lane < nw) sh[lane] = si - s;
        if (lane == nw - 1) sh[31] = si;
    }
    __syncthreads();
    *total = sh[31];
    return sh[w] + incl;
}

// The same scan with ONE block barrier: every warp reads all warp totals after it and forms its
// own offset.  The totals alternate between two buffers (par), so a warp still reading scan i's
// totals cannot see scan i+1's (which completes a barrier all warps pass only after reading).
// The additions are the same as block_incl_scan_d's, in the same order (bitwise equal results).
__device__ __forceinline__ double block_incl_scan_d1(double x, double (*sh)[32], int& par, double* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    double* b = sh[par];
    par ^= 1;
    if (lane == 31) b[w] = incl;
    __syncthreads();
    const double s = (lane < nw) ? b[lane] : 0.0;
    double si = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, si, o);
        if (lane >= o) si += y;
    }
    const double excl = __shfl_sync(0xffffffffu, si - s, w);
    *total = __shfl_sync(0xffffffffu, si, nw - 1);
    return excl + incl;
}

// exclusive prefix of frame fl's (group-local) tile totals of channel c → tileBase (fixed order)
__device__ __forceinline__ void tile_bases(const HierArgs& h, int c, int fl, double* sh) {
    const int t0 = h.tileFrameOff[fl], nt = h.tileFrameOff[fl + 1] - t0;
    const double* agg = h.tileAgg + (size_t)c * h.nTiles1 + t0;
    double* base = h.tileBase + (size_t)c * h.nTiles1 + t0;
    double carry = 0.0;
    for (int b = 0; b < nt; b += blockDim.x) {
        const int tt = b + threadIdx.x;
        const double x = (tt < nt) ? __ldcg(agg + tt) : 0.0;
        double tot;
        const double incl = block_incl_scan_d(x, sh, &tot);
        if (tt < nt) base[tt] = carry + incl - x;
        carry += tot;
    }
}

// PDA: μ_1 = z_w(1) P(1)_1 / (P diagA)_1.
constexpr int kLiftMaxItems = 32;  // (frame, channel) completions a block defers to its end
constexpr int kCoarseTiles = 2048; // tile bases a coarse block scans into shared memory (16 KB)
#ifndef FBS_LIFT_MINB
#define FBS_LIFT_MINB 6  // ≤ 40 registers: 6 blocks per SM (28.6 µs in the step against 36.9 at 62 registers)
#endif
template <int MODE, bool KS = false>
__global__ void __launch_bounds__(kScanTile, FBS_LIFT_MINB) k_tree_lift(HierArgs h, const float* __restrict__ in0,
                                                       const int* __restrict__ active) {
    pdl_entry();
    __shared__ float stage[kScanTile / 32][kLiftStage];
    __shared__ double shs[32];
    __shared__ double shs2[2][32];  // block_incl_scan_d1's warp totals
    int par = 0;
    __shared__ int sfc[kLiftMaxItems];   // (channel, group-local frame) of each finished item
    __shared__ int sdone[kLiftMaxItems]; // 1: this block finished that (frame, channel)'s last tile
    const int tB = h.tileFrameOff[0], nT = h.tileFrameOff[h.nfG] - tB;  // this group's tiles (device)
    const int CW = KS ? h.C : 1;  // KS: channel split (K > 1), one channel per work item
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int nDone = 0;  // items (× channels) of this block whose tile counts are still to be added
    // add this block's finished tiles to their (frame, channel) counters — one atomic per entry, all
    // in flight at once — and scan every frame whose last tile this block finished
    auto settle = [&]() {
        if (threadIdx.x == 0) __threadfence();  // this block's tile totals (written by thread 0)
        __syncthreads();
        if ((int)threadIdx.x < nDone) {
            const int fc = sfc[threadIdx.x], c = fc / h.nfG, fl = fc - c * h.nfG;
            __threadfence();
            unsigned* ctr = h.tcount + (size_t)c * h.F + h.f0 + fl;
            const unsigned nft = (unsigned)(h.tileFrameOff[fl + 1] - h.tileFrameOff[fl]);
            const bool last = atomicAdd(ctr, 1u) == nft - 1u;
            if (last) *ctr = 0u;
            sdone[threadIdx.x] = last;
        }
        __syncthreads();
        for (int e = 0; e < nDone; ++e)
            if (sdone[e]) {
                __threadfence();
                const int fc = sfc[e], c = fc / h.nfG;
                tile_bases(h, c, fc - c * h.nfG, shs);
            }
        __syncthreads();
        nDone = 0;
    };
    for (int item = blockIdx.x; item < nT * CW; item += gridDim.x) {
        const int t = tB + (KS ? item % nT : item);  // global tile id
        const int cB = KS ? item / nT : 0, cE = KS ? cB + 1 : h.C;
        const int fl = h.tileFrame[t] - h.f0;  // group-local frame
        const int2 tr = h.tileRange[t];  // tree positions [i0, i1) of this tile (one frame)
        const int i0 = tr.x, i1 = tr.y;
        const int i = i0 + (int)threadIdx.x;
        const bool valid = i < i1;
        const int wa = min(i0 + 32 * w, i1), wb = min(i0 + 32 * w + 32, i1);
        const int qa = h.csT[wa], qb = h.csT[wb];
        const int myLo = valid ? h.csT[i] : 0, myHi = valid ? h.csT[i + 1] : 0;
        // a frame with more tiles than the coarse kernel scans in shared memory (kCoarseTiles) gets
        // its tile bases from the block that lifts its last tile
        const bool big = h.tileFrameOff[fl + 1] - h.tileFrameOff[fl] > h.coarseTiles;
        for (int c = cB; c < cE; ++c) {
            if (big) {
                if (nDone == kLiftMaxItems) settle();
                if (threadIdx.x == 0) sfc[nDone] = c * h.nfG + fl;
                ++nDone;
            }
            // PCG: a (frame, channel) that has stopped needs no lift (the coarse and level-0
            // passes skip it); its tiles still count towards the frame's scan
            if (MODE == HIER_PCG && active && !active[fl * h.C + c]) continue;
            const float* src = in0 + (size_t)c * h.M0;
            float acc = 0.f;
            for (int qc = qa; qc < qb; qc += kLiftStage) {
                const int n = min(kLiftStage, qb - qc);
                constexpr int E = kLiftStage / 32;
                int id[E];
                float val[E];
#pragma unroll
                for (int e = 0; e < E; ++e) id[e] = (lane + 32 * e < n) ? __ldcs(h.tord0 + qc + lane + 32 * e) : -1;
#pragma unroll
                for (int e = 0; e < E; ++e) val[e] = (id[e] >= 0) ? src[id[e]] : 0.f;
#pragma unroll
                for (int e = 0; e < E; ++e)
                    if (lane + 32 * e < n) stage[w][lane + 32 * e] = val[e];
                __syncwarp();
                const int lo = max(myLo, qc), hi = min(myHi, qc + n);
                for (int q = lo; q < hi; ++q) acc += stage[w][q - qc];
                __syncwarp();
            }
            if (valid) h.buf1T[(size_t)c * h.M1 + i] = acc;
            if (MODE == HIER_PDA && valid)
                h.mu1T[i] = (1 < h.frameLevels[fl] && acc > 0.f) ? zw_count(h, 1, myHi - myLo, (double)acc) : 0.f;
            double tot;
            const double incl = block_incl_scan_d1(valid ? (double)acc : 0.0, shs2, par, &tot);
            if (valid) h.locT[(size_t)c * h.M1 + i] = incl;
            if (threadIdx.x == 0) h.tileAgg[(size_t)c * h.nTiles1 + t] = tot;
        }
    }
    if (__syncthreads_or(nDone > 0)) settle();
}

// ================================================================ coarse values and their projection onto level 2
// Π(j) = fp64 inclusive prefix of tree-ordered (P y)_1 of frame f up to position j: the frame's
// exclusive tile base (k_tree_lift) plus the within-tile prefix; tb = this channel's tile bases
// from the frame's first tile
__device__ __forceinline__ double tree_prefix(const HierArgs& h, const double* tb, int c, int fb, int j) {
    if (j < fb) return 0.0;
    return tb[(j - fb) / kScanTile] + __ldg(h.locT + (size_t)c * h.M1 + j);
}

// One thread per level-2 vertex a (blocks per frame: h.bpf2): (P y)_a and those of its ancestors
// (level-1 ranges and multipliers from the ancestor tables, four per load round), then acc1 for
// its children (L = 2: one thread per level-1 position, acc2 = 0):
//   PCG/PLAIN: acc2_a = Σ_{k≥2} μ_k (P w)_anc;  PCG also ρ_{≥1} = Σ μ (P w)² (each coarse vertex
//              counted once, by its first level-2 descendant; level 1 by its parent) and, in the
//              last block of the frame, the ρ finish (with the ρ_0, ‖r‖² partials of
//              k_hier_level0): β and the stopping rule (Alg. 2 lines 11-13).
//   INIT:      mult_k = z_w(k)/P(1)_k.
// PDA (one thread per coarse vertex of every level ≥ 1... levels ≥ 2 here, level 1 in the lift):
//   μ_k = z_w(k; α, β) P(1)_k / P(diag A)_k, 0 where the denominator is 0
//   (reading #10) or above the frame's top level.
// G = 8 (small problems, api.cu): a group of G lanes per level-2 vertex, lane t taking the levels
// 2 + t, 2 + t + G, …: the ancestor ranges, multipliers and prefix values of all levels go out in
// one round trip each instead of one round per four levels; the fp32 contributions are summed by
// the group's first lane in level order (the same additions as G = 1), the children split over
// the lanes.
template <int MODE, bool KS = false, int G = 1>
__global__ void __launch_bounds__(256) k_tree_coarse(HierArgs h, VecArgs a, int first) {
    pdl_entry();
    __shared__ double shd[32];
    __shared__ int sflag;
    __shared__ double tbS[kCoarseTiles];  // the frame's exclusive tile bases (frames ≤ kCoarseTiles tiles)
    __shared__ double shd2[2][32];
    // KS: channel split (K > 1), grid nf · bpf2 · C, one channel per block group
    const int nfb = KS ? (int)(gridDim.x / h.C) : (int)gridDim.x;
    const int bx = KS ? (int)(blockIdx.x % nfb) : (int)blockIdx.x;
    const int cB = KS ? (int)(blockIdx.x / nfb) : 0, cE = KS ? cB + 1 : h.C;
    const int f = bx / h.bpf2, j = bx % h.bpf2;
    const int F1 = h.F + 1;
    const int fb = h.lvFrameOff[F1 + f];
    const int top = h.L - 1;
    const int fl = h.frameLevels[f];
    const int stride = h.bpf2 * blockDim.x;
    const int lv = (top >= 2) ? 2 : 1;  // level of the threads' vertices
    const int a0 = h.lvFrameOff[lv * F1 + f], a1 = h.lvFrameOff[lv * F1 + f + 1];
    for (int c = cB; c < cE; ++c) {
        const int fk = f * a.K + c;
        const bool act = (MODE != HIER_PCG) || first || a.sc_.active[fk];
        double rho = 0.0;
        if (act) {
            const int t0 = h.tileFrameOff[f], ntf = h.tileFrameOff[f + 1] - t0;
            const double* tb = h.tileBase + (size_t)c * h.nTiles1 + t0;  // big frames: from k_tree_lift
            if (ntf <= h.coarseTiles) {  // scan the frame's tile totals here (fixed order)
                const double* agg = h.tileAgg + (size_t)c * h.nTiles1 + t0;
                double carry = 0.0;
                int par = 0;
                for (int b = 0; b < ntf; b += blockDim.x) {
                    const int tt = b + threadIdx.x;
                    const double x = (tt < ntf) ? agg[tt] : 0.0;
                    double tot;
                    const double incl = block_incl_scan_d1(x, shd2, par, &tot);
                    if (tt < ntf) tbS[tt] = carry + incl - x;
                    carry += tot;
                }
                __syncthreads();
                tb = tbS;
            }
            if (MODE == HIER_PDA) {
                for (int k = 2; k <= top; ++k) {
                    const HLevel& L = h.lv[k];
                    float* mu = const_cast<float*>(L.mu);
                    const int b0 = h.lvFrameOff[k * F1 + f], b1 = h.lvFrameOff[k * F1 + f + 1];
                    for (int v = b0 + j * blockDim.x + threadIdx.x; v < b1; v += stride) {
                        const int2 rg = L.rng[v];
                        const double S = tree_prefix(h, tb, c, fb, rg.x + rg.y - 1) - tree_prefix(h, tb, c, fb, rg.x - 1);
                        mu[v] = (k < fl && S > 0.0) ? zw_count(h, k, L.count[v], S) : 0.f;
                    }
                }
                continue;
            }
            if constexpr (G > 1) {
                const int lane = threadIdx.x & 31, t = lane % G, gl0 = lane - t;
                const int gpb = blockDim.x / G;  // vertex groups per block
                for (int vb = a0 + j * gpb; vb < a1; vb += h.bpf2 * gpb) {  // uniform over the block
                    const int v = vb + (int)threadIdx.x / G;
                    const bool valid = v < a1;
                    const int2 kids = valid ? h.lv[2].rng[v] : make_int2(0, 0);
                    const int first1 = kids.x;
                    float acc = 0.f;
                    for (int kb = 2; kb <= top; kb += G) {  // levels kb + t of every lane
                        const int k = kb + t;
                        float cv = 0.f;
                        if (valid && k <= top) {
                            int2 r;
                            float m;
                            if (k == 2) {
                                r = kids;
                                m = (MODE == HIER_INIT) ? init_mult1(h, 2, fl, h.lv[2].count[v]) : h.lv[2].mu[v];
                            } else {
                                const size_t o = (size_t)(k - 3) * h.M2 + v;
                                r = __ldg(h.ancRng + o);
                                m = __ldg(h.ancMult + o);
                            }
                            const double S = tree_prefix(h, tb, c, fb, r.x + r.y - 1) - tree_prefix(h, tb, c, fb, r.x - 1);
                            cv = m * (float)S;
                            if (MODE == HIER_PCG && (k == 2 || r.x == first1)) rho += (double)m * S * S;
                        }
                        // the group's first lane adds the levels in order (as the G = 1 loop does)
#pragma unroll
                        for (int u = 0; u < G; ++u) {
                            const float cu = __shfl_sync(0xffffffffu, cv, gl0 + u);
                            if (u == 0 && kb == 2) acc = cu;
                            else if (kb + u <= top) acc += cu;
                        }
                    }
                    acc = __shfl_sync(0xffffffffu, acc, gl0);
                    // acc1 for the children, split over the group's lanes
                    const float* b1 = h.buf1T + (size_t)c * h.M1;
                    for (int i = kids.x + t; valid && i < kids.x + kids.y; i += G) {
                        const float m1 = (MODE == HIER_INIT) ? init_mult1(h, 1, fl, h.csT[i + 1] - h.csT[i]) : h.mu1T[i];
                        const float bv = b1[i];
                        h.acc1T[(size_t)c * h.M1 + i] = m1 * bv + acc;
                        if (MODE == HIER_PCG) rho += (double)m1 * (double)bv * (double)bv;
                    }
                }
            } else
            for (int v = a0 + j * blockDim.x + threadIdx.x; v < a1; v += stride) {
                // level-1 children of v: one contiguous tree range (L = 2: v itself)
                const int2 kids = (lv == 2) ? h.lv[2].rng[v] : make_int2(v, 1);
                const int first1 = kids.x;
                float acc = 0.f;
                if (lv == 2) {
                    {   // v itself
                        const double S = tree_prefix(h, tb, c, fb, kids.x + kids.y - 1) - tree_prefix(h, tb, c, fb, kids.x - 1);
                        const float m = (MODE == HIER_INIT) ? init_mult1(h, 2, fl, h.lv[2].count[v]) : h.lv[2].mu[v];
                        acc = m * (float)S;
                        if (MODE == HIER_PCG) rho += (double)m * S * S;
                    }
                    for (int kb = 3; kb <= top; kb += 4) {  // its ancestors, four per load round
                        int2 r[4];
                        float m[4];
                        double S[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            if (kb + u > top) continue;
                            const size_t o = (size_t)(kb + u - 3) * h.M2 + v;
                            r[u] = __ldg(h.ancRng + o);
                            m[u] = __ldg(h.ancMult + o);
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (kb + u <= top)
                                S[u] = tree_prefix(h, tb, c, fb, r[u].x + r[u].y - 1) - tree_prefix(h, tb, c, fb, r[u].x - 1);
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            if (kb + u > top) continue;
                            acc += m[u] * (float)S[u];
                            if (MODE == HIER_PCG && r[u].x == first1) rho += (double)m[u] * S[u] * S[u];
                        }
                    }
                }
                // acc1 for the children (+ PCG: their ρ_1 terms μ_1 (P w)²_1), 4 loads in flight
                const float* b1 = h.buf1T + (size_t)c * h.M1;
                for (int ib = kids.x; ib < kids.x + kids.y; ib += 4) {
                    float m1[4], bv[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int i = ib + u;
                        if (i < kids.x + kids.y) {
                            m1[u] = (MODE == HIER_INIT) ? init_mult1(h, 1, fl, h.csT[i + 1] - h.csT[i]) : h.mu1T[i];
                            bv[u] = b1[i];
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int i = ib + u;
                        if (i < kids.x + kids.y) {
                            h.acc1T[(size_t)c * h.M1 + i] = m1[u] * bv[u] + acc;
                            if (MODE == HIER_PCG) rho += (double)m1[u] * (double)bv[u] * (double)bv[u];
                        }
                    }
                }
            }
        }
        if (MODE == HIER_PCG) {
            rho = block_sum(rho, shd);
            if (threadIdx.x == 0) h.partial2[((size_t)f * h.bpf2 + j) * h.C + c] = rho;
        }
    }
    if (MODE == HIER_PCG && last_block_t0(h.counters + (KS ? (size_t)cB * h.F : 0) + f, h.bpf2, &sflag)) {
        for (int c = (KS ? cB : 0); c < (KS ? cE : a.K); ++c) {
            const int fk = f * a.K + c;
            if (!first && !a.sc_.active[fk]) continue;
            double R = 0.0, RR = 0.0;
            for (int jj = threadIdx.x; jj < a.BPF; jj += blockDim.x) {
                const double* pp = a.partial + ((size_t)f * a.BPF + jj) * 2 * a.K + 2 * c;
                R += __ldcg(pp);
                RR += __ldcg(pp + 1);
            }
            for (int jj = threadIdx.x; jj < h.bpf2; jj += blockDim.x)
                R += __ldcg(h.partial2 + ((size_t)f * h.bpf2 + jj) * h.C + c);
            block_sum2(R, RR, shd);
            if (threadIdx.x == 0) finish_rho_one(a, fk, first != 0, R, RR);
            __syncthreads();
        }
    }
}

// ================================================================ level 0
// acc1 = acc1T at the tree position pT of the level-1 parent, then
// PCG:   d = s + βd with s = mask∘(μ0 r + acc1) (Alg. 2 line 14; first: d = s, line 3)
// PLAIN: out0 = mask∘(μ0 in0 + acc1[parent])
// INIT:  out0_k = (in0_k + acc1_k[parent]) / (in0_K + acc1_K[parent]), 0 where the denominator is 0
template <int MODE, bool KS = false>
__global__ void __launch_bounds__(256) k_tree_level0(HierArgs h, VecArgs a, const float* __restrict__ in0,
                                                   float* __restrict__ out0, int first) {
    pdl_entry();
    int f, j, kB, kE, ci;  // frame, part, channels [kB, kE), last-block counter index
    if constexpr (KS) {    // channel split (K > 1): one (frame, channel) per block group
        const int g = blockIdx.x / a.BPF;
        j = blockIdx.x - g * a.BPF;
        f = g / a.K;
        kB = g - f * a.K;
        kE = kB + 1;
        ci = g;
    } else {
        f = blockIdx.x / a.BPF;
        j = blockIdx.x % a.BPF;
        kB = 0;
        kE = a.K;
        ci = f;
    }
    const int v0 = a.frameOff[f], v1 = a.frameOff[f + 1];
    const int stride = a.BPF * blockDim.x;
    const int K = (MODE == HIER_INIT) ? h.C - 1 : a.K;
    auto acc1 = [&](int c, int pT) { return h.acc1T[(size_t)c * h.M1 + pT]; };
    for (int k = KS ? kB : 0; k < (KS ? kE : K); ++k) {
        const int fk = f * a.K + k;
        // PCG: this iteration's x += αd (Alg. 2 line 8, deferred from the update kernel) for every
        // channel the SpMV advanced, even one that stopped since; the new direction for active ones
        const float xa = (MODE == HIER_PCG && !first) ? (float)a.sc_.xalpha[fk] : 0.f;
        const bool dir = MODE != HIER_PCG || first || a.sc_.active[fk];
        if (!dir && xa == 0.f) continue;
        const float be = (MODE == HIER_PCG && !first) ? (float)a.sc_.beta[fk] : 0.f;
        const size_t off = (size_t)k * a.M;
        for (int vb = v0 + j * blockDim.x + threadIdx.x; vb < v1; vb += kL0B * stride) {
            float sv[kL0B], mv[kL0B], up[kL0B], xv[kL0B];
            float2 dv[kL0B];
#pragma unroll
            for (int u = 0; u < kL0B; ++u) {
                const int v = vb + u * stride;
                if (v < v1) {
                    const int pT = __ldcs(h.parent0T + v);
                    up[u] = acc1(k, pT);
                    if (MODE == HIER_INIT) {
                        sv[u] = in0[off + v];
                        mv[u] = in0[(size_t)K * a.M + v] + acc1(K, pT);
                    } else {
                        sv[u] = (MODE == HIER_PCG) ? __ldcs(a.r + off + v) : in0[off + v];
                        mv[u] = __ldcs(a.mu0 + v);
                        if (MODE == HIER_PCG) {
                            dv[u] = a.dn[(size_t)k * a.ldn + v];
                            if (xa != 0.f) xv[u] = a.x[off + v];
                        }
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < kL0B; ++u) {
                const int v = vb + u * stride;
                if (v >= v1) continue;
                if (MODE == HIER_INIT) {
                    out0[off + v] = (mv[u] > 0.f) ? (sv[u] + up[u]) / mv[u] : 0.f;
                } else {
                    const float s = (mv[u] > 0.f) ? mv[u] * sv[u] + up[u] : 0.f;
                    if (MODE == HIER_PCG) {
                        if (xa != 0.f) a.x[off + v] = xv[u] + xa * dv[u].x;
                        if (dir) a.dn[(size_t)k * a.ldn + v] = make_float2(first ? s : s + be * dv[u].x, dv[u].y);
                    } else {
                        out0[off + v] = s;
                    }
                }
            }
        }
    }
}

}  // namespace fbs
