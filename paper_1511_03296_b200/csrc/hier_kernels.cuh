// hier_kernels.cuh — the hierarchical preconditioner and initialisation kept on-chip
// (Eq. hier_precond, hier init PAPER.md:287-293, pyramid PAPER.md:745-766).
//
// P(y) lifts bottom-up and Pᵀ(z) projects top-down through the pyramid.  Both are tree
// operations: a level-(k+1) vertex's children live in the ≤2×2 level-k cells under its own
// cell.  So the subtree of every level-T vertex lies inside one level-T cell ("tile" = 2^T × 2^T
// base cells).  One CTA per tile does the levels 0..T part of the lift (fused with the PCG update
// that produces the level-0 input) and, later, the levels T..0 part of the projection (fused with
// the level-0 combination s = mask∘(μ0 w + …) and the ρ = rᵀs reduction), entirely in shared
// memory.  Only levels ≥ T — a few thousand vertices per frame — go through global memory, in one
// small per-frame kernel.  Every sum runs over the child lists in canonical order, so results are
// deterministic.
#pragma once
#include "fbs_common.cuh"
#include "solve_kernels.cuh"

namespace fbs {

// ---------------------------------------------------------------- tile geometry (shared memory)
struct ProgOff {
    int seg[kTileT + 1], ch[kTileT + 1], par[kTileT + 1], total;
};

struct TileRuns {
    int start[kTileT + 1][kTileRows];
    int len[kTileT + 1][kTileRows];
    int off[kTileT + 1][kTileRows + 1];
    int rows[kTileT + 1];
    int cpre[kTileT + 1][kTileRows + 1];  // 32-element chunk prefix per row (chunked loops)
    ProgOff po;  // tile-program offsets (see "tile programs" below)
};

__device__ __forceinline__ void tile_runs(const HierArgs& h, int f, int TY, int TX, TileRuns& tr) {
    // thread t < (T+1)·8 fills run (k, j)
    const int t = threadIdx.x;
    if (t < (h.T + 1) * kTileRows) {
        const int k = t / kTileRows, j = t % kTileRows;
        const int R = 1 << (h.T - k);
        const HLevel& L = h.lv[k];
        const int cy = TY * R + j;
        const int cx0 = TX * R, cx1 = min(TX * R + R, L.ncx);
        int st = 0, ln = 0;
        if (j < R && cy < L.ncy && cx0 < cx1) {
            const int64_t c0 = ((int64_t)f * L.ncy + cy) * L.ncx + cx0;
            st = L.cellOff[c0];
            ln = L.cellOff[c0 + (cx1 - cx0)] - st;
        }
        tr.start[k][j] = st;
        tr.len[k][j] = ln;
    }
    __syncthreads();
    if (t <= h.T) {
        int acc = 0, cacc = 0;
        const int R = 1 << (h.T - t);
        tr.off[t][0] = 0;
        tr.cpre[t][0] = 0;
        for (int j = 0; j < kTileRows; ++j) {
            const int ln = (j < R) ? tr.len[t][j] : 0;
            acc += ln;
            cacc += (ln + 31) >> 5;
            tr.off[t][j + 1] = acc;
            tr.cpre[t][j + 1] = cacc;
        }
        tr.rows[t] = R;
    }
    __syncthreads();
    if (t == 0) {
        int off = 0;
        for (int k = 1; k <= h.T; ++k) {
            tr.po.seg[k] = off;
            off += tr.off[k][tr.rows[k]] + 1;
            tr.po.ch[k] = off;
            off += tr.off[k - 1][tr.rows[k - 1]];
        }
        for (int k = 0; k < h.T; ++k) {
            tr.po.par[k] = off;
            off += tr.off[k][tr.rows[k]];
        }
        tr.po.total = off;
    }
    __syncthreads();
}

// local index i (level k) → (row j, global id g)
__device__ __forceinline__ int tile_global(const TileRuns& tr, int k, int i, int& j) {
    j = 0;
    while (i >= tr.off[k][j + 1]) ++j;
    return tr.start[k][j] + (i - tr.off[k][j]);
}

// global id g known to lie in level-k row j0 or j0+1 → local index
__device__ __forceinline__ int tile_local2(const TileRuns& tr, int k, int g, int j0) {
    const int j = (g >= tr.start[k][j0] && g < tr.start[k][j0] + tr.len[k][j0]) ? j0 : j0 + 1;
    return tr.off[k][j] + (g - tr.start[k][j]);
}

// lift level k → k+1 inside the tile: vals[k+1][i'] = Σ children vals[k][·]
__device__ __forceinline__ void tile_lift_level(const HierArgs& h, const TileRuns& tr, int k, const float* src,
                                                float* dst, float* gout /* buf_{k+1} channel row or null */) {
    const HLevel& Lu = h.lv[k + 1];
    const int n = tr.off[k + 1][tr.rows[k + 1]];
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        int j;
        const int p = tile_global(tr, k + 1, i, j);
        float acc = 0.f;
        for (int q = Lu.childStart[p]; q < Lu.childStart[p + 1]; ++q)
            acc += src[tile_local2(tr, k, Lu.childList[q], 2 * j)];
        dst[i] = acc;
        if (gout) gout[p] = acc;
    }
}


// ---------------------------------------------------------------- tile programs
// The pyramid's structure inside a tile, precompiled once per grid in tile-local u16 indices
// (all < kTileCap) and stored contiguously per tile, so the per-iteration lifts and projections
// touch only shared memory.  Layout (u16), n_k = the tile's level-k vertex count:
//   [seg_1 (n1+1)][ch_1 (n0)] … [seg_T (nT+1)][ch_T (n_{T−1})][par_0 (n0)] … [par_{T−1} (n_{T−1})]
// seg_k/ch_k: children (level-k−1 local ids) of each level-k vertex in canonical child order;
// par_k: local id of each level-k vertex's parent at level k+1.
// capacity (u16 entries, even) of one tile's program from the per-level maxima
inline int prog_capacity(const int* tm, int T) {
    int c = 0;
    for (int k = 1; k <= T; ++k) c += tm[k] + 1 + tm[k - 1];
    for (int k = 0; k < T; ++k) c += tm[k];
    return (c + 1) & ~1;
}

__global__ void __launch_bounds__(256) k_tile_program(HierArgs h, int cap, uint16_t* __restrict__ prog) {
    __shared__ TileRuns tr;
    __shared__ int rowChildOff[kTileT + 1][kTileRows];
    const int tile = blockIdx.x;
    const int per = h.ntx * h.nty;
    const int f = tile / per, TY = (tile % per) / h.ntx, TX = tile % h.ntx;
    tile_runs(h, f, TY, TX, tr);
    if (threadIdx.x >= 1 && threadIdx.x <= h.T) {
        const int k = threadIdx.x;
        int acc = 0;
        for (int j = 0; j < tr.rows[k]; ++j) {
            rowChildOff[k][j] = acc;
            if (tr.len[k][j] > 0)
                acc += h.lv[k].childStart[tr.start[k][j] + tr.len[k][j]] - h.lv[k].childStart[tr.start[k][j]];
        }
    }
    __syncthreads();
    const ProgOff& o = tr.po;
    uint16_t* P = prog + (size_t)tile * cap;
    for (int k = 1; k <= h.T; ++k) {
        const HLevel& L = h.lv[k];
        const int n = tr.off[k][tr.rows[k]];
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            int j;
            const int p = tile_global(tr, k, i, j);
            const int cs = L.childStart[p], ce = L.childStart[p + 1];
            const int seg = rowChildOff[k][j] + (cs - L.childStart[tr.start[k][j]]);
            P[o.seg[k] + i] = (uint16_t)seg;
            if (i == n - 1) P[o.seg[k] + n] = (uint16_t)(seg + (ce - cs));
            for (int q = cs; q < ce; ++q)
                P[o.ch[k] + seg + (q - cs)] = (uint16_t)tile_local2(tr, k - 1, L.childList[q], 2 * j);
        }
    }
    for (int k = 0; k < h.T; ++k) {
        const int n = tr.off[k][tr.rows[k]];
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            int j;
            const int g = tile_global(tr, k, i, j);
            P[o.par[k] + i] = (uint16_t)tile_local2(tr, k + 1, h.lv[k].parent[g], j >> 1);
        }
    }
}

enum { UP_PCG = 0, UP_PLAIN = 1 };

// ---------------------------------------------------------------- chunked tile loops
// A tile's level-k vertices are a few row runs (contiguous in memory).  Loops walk them in
// chunks of 32 consecutive elements of one row: a warp takes whole chunks (coalesced, no
// per-element row search), the row cursor is warp-uniform and advances monotonically, and
// U chunks' loads are issued before any of them is used (memory-level parallelism; the
// VecArgs pointers may alias as far as the compiler knows, so loads are hoisted by hand).
__device__ __forceinline__ int chunk_row(const int* cpre, int r, int c) {
    while (c >= cpre[r + 1]) ++r;
    return r;
}

template <int U, class LD, class ST>
__device__ __forceinline__ void stage_unrolled(int n, LD ld, ST st) {
    for (int i0 = threadIdx.x; i0 < n; i0 += U * blockDim.x) {
        decltype(ld(0)) v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * blockDim.x;
            if (i < n) v[u] = ld(i);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * blockDim.x;
            if (i < n) st(i, v[u]);
        }
    }
}

// ---------------------------------------------------------------- up: level 0 → T
// w = in[c] (masked to live vertices if `mask_in`), c < C  (UP_PLAIN; the PCG update that
// produces w runs vertex-parallel in k_update<true>).
// Lifts w through levels 1..T in shared memory with the tile program and writes
// the lifted values to the global level buffers (level T feeds the coarse kernel, levels 1..T−1
// the projection).
template <int MODE>
__global__ void __launch_bounds__(256) k_tile_up(HierArgs h, VecArgs a, const float* __restrict__ in, int mask_in) {
    extern __shared__ float sv[];  // level arrays at h.soff[k], then the tile program (u16)
    __shared__ TileRuns tr;
    const int tile = blockIdx.x;
    const int per = h.ntx * h.nty;
    const int f = tile / per, TY = (tile % per) / h.ntx, TX = tile % h.ntx;
    tile_runs(h, f, TY, TX, tr);
    const ProgOff& o = tr.po;
    uint16_t* sp = reinterpret_cast<uint16_t*>(sv + h.soff[h.T + 1]);
    {   // stage the lift part of the program (seg/ch of levels 1..T)
        const unsigned* src = reinterpret_cast<const unsigned*>(h.prog + (size_t)tile * h.progCap);
        unsigned* dst = reinterpret_cast<unsigned*>(sp);
        const int nw = (o.par[0] + 1) >> 1;
        stage_unrolled<4>(nw, [&](int i) { return __ldg(src + i); }, [&](int i, unsigned v) { dst[i] = v; });
    }
    const int nwarp = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int c = 0; c < h.C; ++c) {
        const size_t off = (size_t)c * a.M;
        const int nc0 = tr.cpre[0][tr.rows[0]];
        int r = 0;
        for (int c0 = warp; c0 < nc0; c0 += 4 * nwarp) {
            int gg[4], li[4];
            float rv[4], mv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int cc = c0 + u * nwarp;
                gg[u] = -1;
                if (cc < nc0) {
                    r = chunk_row(tr.cpre[0], r, cc);
                    const int e = ((cc - tr.cpre[0][r]) << 5) + lane;
                    if (e < tr.len[0][r]) {
                        const int g = tr.start[0][r] + e;
                        gg[u] = g;
                        li[u] = tr.off[0][r] + e;
                        rv[u] = in[off + g];
                        mv[u] = a.mu0[g];
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int g = gg[u];
                if (g < 0) continue;
                const float w = (mask_in && !(mv[u] > 0.f)) ? 0.f : rv[u];
                sv[li[u]] = w;
            }
        }
        __syncthreads();
        for (int k = 1; k <= h.T; ++k) {
            const float* src = sv + h.soff[k - 1];
            float* dst = sv + h.soff[k];
            const HLevel& Lk = h.lv[k];
            float* gout = Lk.buf + (size_t)c * Lk.M;
            const uint16_t* seg = sp + o.seg[k];
            const uint16_t* ch = sp + o.ch[k];
            const int nck = tr.cpre[k][tr.rows[k]];
            int rk = 0;
            for (int cc = warp; cc < nck; cc += nwarp) {
                rk = chunk_row(tr.cpre[k], rk, cc);
                const int e = ((cc - tr.cpre[k][rk]) << 5) + lane;
                if (e < tr.len[k][rk]) {
                    const int i = tr.off[k][rk] + e;
                    float acc = 0.f;
                    const int q1 = seg[i + 1];
#pragma unroll 4
                    for (int q = seg[i]; q < q1; ++q) acc += src[ch[q]];
                    dst[i] = acc;
                    gout[tr.start[k][rk] + e] = acc;
                }
            }
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------- coarse levels T..L−1 (per frame)
// Lift T → top, then project top → T in place:  buf_k = mult_k ∘ buf_k + buf_{k+1}[parent]
// (Pᵀ).  mult_k = μ_k (USE_MU) or z_w(k)/P(1)_k (init), 0 on levels a frame lacks.
__device__ __forceinline__ float level_mult(const HierArgs& h, int k, int v, int f, bool use_mu) {
    if (use_mu) return h.lv[k].mu[v];
    if (k >= h.frameLevels[f]) return 0.f;
    const double zw = (k == 0) ? 1.0 : pow(h.alpha, -(h.beta + (double)k));
    return (float)(zw / (double)h.lv[k].count[v]);
}

__global__ void __launch_bounds__(1024) k_coarse(HierArgs h, int use_mu, int do_project) {
    const int f = blockIdx.x;
    const int top = h.L - 1;
    for (int c = 0; c < h.C; ++c) {
        for (int k = h.T; k < top; ++k) {  // lift k → k+1 over the frame's level-(k+1) vertices
            const HLevel& Lu = h.lv[k + 1];
            const float* src = h.lv[k].buf + (size_t)c * h.lv[k].M;
            float* dst = Lu.buf + (size_t)c * Lu.M;
            const int v0 = h.lvFrameOff[(k + 1) * (h.F + 1) + f], v1 = h.lvFrameOff[(k + 1) * (h.F + 1) + f + 1];
            for (int p = v0 + threadIdx.x; p < v1; p += blockDim.x) {
                float acc = 0.f;
                for (int q = Lu.childStart[p]; q < Lu.childStart[p + 1]; ++q) acc += src[Lu.childList[q]];
                dst[p] = acc;
            }
            __syncthreads();
        }
        if (!do_project) continue;
        for (int k = top; k >= h.T; --k) {
            const HLevel& L = h.lv[k];
            float* b = L.buf + (size_t)c * L.M;
            const float* up = (k < top) ? h.lv[k + 1].buf + (size_t)c * h.lv[k + 1].M : nullptr;
            const int v0 = h.lvFrameOff[k * (h.F + 1) + f], v1 = h.lvFrameOff[k * (h.F + 1) + f + 1];
            for (int v = v0 + threadIdx.x; v < v1; v += blockDim.x) {
                float val = level_mult(h, k, v, f, use_mu != 0) * b[v];
                if (up) val += up[L.parent[v]];
                b[v] = val;
            }
            __syncthreads();
        }
    }
}


// Shared-memory variant of k_coarse: the frame's whole coarse pyramid (levels T..top: child
// lists, parents, multipliers, values) is staged with one burst of independent loads, then
// every level is lifted and projected in shared memory.  Used when it fits (api.cu sizes it).
__global__ void __launch_bounds__(512) k_coarse_smem(HierArgs h, int use_mu, int do_project) {
    extern __shared__ float cs_smem[];
    const int f = blockIdx.x;
    const int T = h.T, top = h.L - 1, F1 = h.F + 1;
    // frame-local level ranges and the shared-memory carve-up
    __shared__ int v0[kMaxLevels], cnt[kMaxLevels], oval[kMaxLevels], omul[kMaxLevels], opar[kMaxLevels],
        ocst[kMaxLevels], ocl[kMaxLevels];
    if (threadIdx.x == 0) {
        int off = 0;
        for (int k = T; k <= top; ++k) {
            v0[k] = h.lvFrameOff[k * F1 + f];
            cnt[k] = h.lvFrameOff[k * F1 + f + 1] - v0[k];
        }
        for (int k = T; k <= top; ++k) {
            oval[k] = off; off += cnt[k];
            omul[k] = off; off += cnt[k];
            opar[k] = off; off += (k < top) ? cnt[k] : 0;
            ocst[k] = off; off += (k > T) ? cnt[k] + 1 : 0;
            ocl[k] = off; off += (k > T) ? cnt[k - 1] : 0;
        }
    }
    __syncthreads();
    float* sf = cs_smem;
    int* si = reinterpret_cast<int*>(cs_smem);
    // structure (channel independent)
    for (int k = T; k <= top; ++k) {
        const HLevel& L = h.lv[k];
        const int base = v0[k];
        if (do_project)
            stage_unrolled<8>(cnt[k], [&](int i) { return level_mult(h, k, base + i, f, use_mu != 0); },
                              [&](int i, float v) { sf[omul[k] + i] = v; });
        if (k < top) {
            const int pb = v0[k + 1];
            stage_unrolled<8>(cnt[k], [&](int i) { return L.parent[base + i] - pb; },
                              [&](int i, int v) { si[opar[k] + i] = v; });
        }
        if (k > T) {
            const int c0 = L.childStart[base];
            const int cb = v0[k - 1];
            stage_unrolled<8>(cnt[k] + 1, [&](int i) { return L.childStart[base + i] - c0; },
                              [&](int i, int v) { si[ocst[k] + i] = v; });
            stage_unrolled<8>(cnt[k - 1], [&](int i) { return L.childList[c0 + i] - cb; },
                              [&](int i, int v) { si[ocl[k] + i] = v; });
        }
    }
    for (int c = 0; c < h.C; ++c) {
        {
            const float* b = h.lv[T].buf + (size_t)c * h.lv[T].M + v0[T];
            stage_unrolled<8>(cnt[T], [&](int i) { return b[i]; }, [&](int i, float v) { sf[oval[T] + i] = v; });
        }
        __syncthreads();
        for (int k = T + 1; k <= top; ++k) {  // lift
            for (int p = threadIdx.x; p < cnt[k]; p += blockDim.x) {
                float acc = 0.f;
                const int q1 = si[ocst[k] + p + 1];
                for (int q = si[ocst[k] + p]; q < q1; ++q) acc += sf[oval[k - 1] + si[ocl[k] + q]];
                sf[oval[k] + p] = acc;
                if (!do_project) h.lv[k].buf[(size_t)c * h.lv[k].M + v0[k] + p] = acc;
            }
            __syncthreads();
        }
        if (!do_project) continue;
        for (int k = top; k >= T; --k) {  // project
            for (int v = threadIdx.x; v < cnt[k]; v += blockDim.x) {
                float val = sf[omul[k] + v] * sf[oval[k] + v];
                if (k < top) val += sf[oval[k + 1] + si[opar[k] + v]];
                sf[oval[k] + v] = val;
                if (k == T) h.lv[T].buf[(size_t)c * h.lv[T].M + v0[T] + v] = val;
            }
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------- project: level T → 1
// Pᵀ inside the tile: acc_k = mult_k ∘ L_k + acc_{k+1}[parent] for k = T−1..1 in
// shared memory (level T was projected by k_coarse), then acc_1 is written back in place to the
// level-1 buffer, where the level-0 combination (k_precond_finish2 / k_init_finish /
// k_precond_out) gathers it through the parent map.  mult_k = μ_k (USE_MU) or z_w(k)/P(1)_k.
template <bool USE_MU>
__global__ void __launch_bounds__(256) k_tile_project(HierArgs h) {
    extern __shared__ float sv[];  // level arrays at h.soff[k]
    __shared__ TileRuns tr;
    const int tile = blockIdx.x;
    const int per = h.ntx * h.nty;
    const int f = tile / per, tj = tile % per, TY = tj / h.ntx, TX = tj % h.ntx;
    tile_runs(h, f, TY, TX, tr);
    const ProgOff& o = tr.po;
    const uint16_t* P = h.prog + (size_t)tile * h.progCap;
    const int nwarp = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int c = 0; c < h.C; ++c) {
        for (int k = h.T; k >= 1; --k) {
            const HLevel& L = h.lv[k];
            float* b = L.buf + (size_t)c * L.M;
            const int nck = tr.cpre[k][tr.rows[k]];
            int rk = 0;
            for (int cc = warp; cc < nck; cc += nwarp) {
                rk = chunk_row(tr.cpre[k], rk, cc);
                const int e = ((cc - tr.cpre[k][rk]) << 5) + lane;
                if (e < tr.len[k][rk]) {
                    const int i = tr.off[k][rk] + e;
                    const int g = tr.start[k][rk] + e;
                    float v;
                    if (k == h.T)
                        v = b[g];
                    else
                        v = level_mult(h, k, g, f, USE_MU) * b[g] + sv[h.soff[k + 1] + P[o.par[k] + i]];
                    sv[h.soff[k] + i] = v;
                    if (k == 1 && h.T > 1) b[g] = v;
                }
            }
            __syncthreads();
        }
    }
}

// Largest per-level vertex count of any level-T tile (sizes the tiles' shared memory).
__global__ void k_tile_maxcounts(HierArgs h, int ntiles, int* __restrict__ out) {
    for (int tile = blockIdx.x * blockDim.x + threadIdx.x; tile < ntiles; tile += gridDim.x * blockDim.x) {
        const int per = h.ntx * h.nty;
        const int f = tile / per, TY = (tile % per) / h.ntx, TX = tile % h.ntx;
        for (int k = 0; k <= h.T; ++k) {
            const int R = 1 << (h.T - k);
            const HLevel& L = h.lv[k];
            int tot = 0;
            for (int j = 0; j < R; ++j) {
                const int cy = TY * R + j;
                const int cx0 = TX * R, cx1 = min(TX * R + R, L.ncx);
                if (cy < L.ncy && cx0 < cx1) {
                    const int64_t c0 = ((int64_t)f * L.ncy + cy) * L.ncx + cx0;
                    tot += L.cellOff[c0 + (cx1 - cx0)] - L.cellOff[c0];
                }
            }
            atomicMax(out + k, tot);
        }
    }
}

}  // namespace fbs

namespace fbs {

// ================================================================ cooperative hierarchy
// One persistent cooperative kernel applies the whole pyramid: each level is one grid-wide
// parallel phase (all frames at once), separated by a grid barrier, so every level uses the
// whole GPU and no launch sits between levels.  Lift P: buf_{k+1}[p] = Σ children
// buf_k in canonical child order; project Pᵀ: buf_k = mult_k∘buf_k +
// buf_{k+1}[parent_k]; then the level-0 phase (mode dependent).  Blocks are assigned per frame
// (blockIdx = f·bpf + j) so the level-0 phase can finish per-frame reductions.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> cnt(bar[0]), gen(bar[1]);
        const unsigned g = gen.load(cuda::memory_order_acquire);
        if (cnt.fetch_add(1u, cuda::memory_order_acq_rel) == nblocks - 1) {
            cnt.store(0u, cuda::memory_order_relaxed);
            gen.store(g + 1, cuda::memory_order_release);
        } else {
            while (gen.load(cuda::memory_order_acquire) == g) __nanosleep(32);
        }
    }
    __syncthreads();
}

enum { HIER_PCG = 0, HIER_PDA = 1, HIER_INIT = 2, HIER_PLAIN = 3 };

// mode  level-0 input (in0)     project        level-0 phase
// PCG   w0 = mask∘r             μ_k            s = mask∘(μ0 r + acc1[parent0]); ρ, ‖r‖²; finish_rho
// PDA   diag(A)∘mask            —              μ_k = z_w(k)·P(1)_k / P(diag A)_k for k ≥ 1
// INIT  [b_0..b_{K−1}, Sc]      z_w(k)/P(1)_k  y0 = num/den (0 where den = 0)
// PLAIN mask∘r (planar)         μ_k            out = mask∘(μ0 r + acc1[parent0])
template <int MODE>
__global__ void __launch_bounds__(1024) k_hier(HierArgs h, VecArgs a, const float* __restrict__ in0,
                                              float* __restrict__ out0, int first, int bpf, unsigned* bar,
                                              int k_lift0, int do_level0) {
    __shared__ double shd[32];
    __shared__ int sflag;
    const unsigned nb = gridDim.x;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
    const int top = h.L - 1;
    const int C = h.C;
    // Levels below kc run as grid-wide phases; levels kc..top of frame f are done by block f
    // alone (a few thousand vertices: no grid barrier per level), between two grid barriers.
    const int kc = min(top, 3);
    auto lift_level = [&](int k, int64_t p_begin, int64_t p_end, int64_t t0, int64_t tstride) {
        const HLevel& Lu = h.lv[k + 1];
        const float* src = (k == 0) ? in0 : h.lv[k].buf;
        const int64_t Msrc = h.lv[k].M;
        for (int64_t p = p_begin + t0; p < p_end; p += tstride) {
            const int q0 = Lu.childStart[p], q1 = Lu.childStart[p + 1];
            for (int c = 0; c < C; ++c) {
                const float* sc = src + (size_t)c * Msrc;
                float acc = 0.f;
                for (int q = q0; q < q1; ++q) acc += sc[Lu.childList[q]];
                Lu.buf[(size_t)c * Lu.M + p] = acc;
            }
        }
    };
    auto project_level = [&](int k, int64_t v_begin, int64_t v_end, int64_t t0, int64_t tstride) {
        const HLevel& L = h.lv[k];
        const float* up = (k < top) ? h.lv[k + 1].buf : nullptr;
        const int64_t Mup = (k < top) ? h.lv[k + 1].M : 0;
        for (int64_t v = v_begin + t0; v < v_end; v += tstride) {
            float mult;
            if (MODE != HIER_INIT) {
                mult = L.mu[v];
            } else {
                const int f = (int)(L.keys[v] >> 56);
                mult = (k < h.frameLevels[f]) ? (float)(pow(h.alpha, -(h.beta + (double)k)) / (double)L.count[v]) : 0.f;
            }
            const int pa = up ? L.parent[v] : 0;
            for (int c = 0; c < C; ++c) {
                float val = mult * L.buf[(size_t)c * L.M + v];
                if (up) val += up[(size_t)c * Mup + pa];
                L.buf[(size_t)c * L.M + v] = val;
            }
        }
    };
    // ---- lift k_lift0 → kc (grid-wide)
    for (int k = k_lift0; k < kc; ++k) {
        lift_level(k, 0, h.lv[k + 1].M, gtid, gstride);
        grid_barrier(bar, nb);
    }
    // ---- levels kc..top per frame (block f), lift then (unless PDA) project
    if ((int)blockIdx.x < h.F) {
        const int f = blockIdx.x, F1 = h.F + 1;
        for (int k = kc; k < top; ++k) {
            lift_level(k, h.lvFrameOff[(k + 1) * F1 + f], h.lvFrameOff[(k + 1) * F1 + f + 1], threadIdx.x,
                       blockDim.x);
            __syncthreads();
        }
        if (MODE != HIER_PDA) {
            for (int k = top; k >= kc; --k) {
                project_level(k, h.lvFrameOff[k * F1 + f], h.lvFrameOff[k * F1 + f + 1], threadIdx.x, blockDim.x);
                __syncthreads();
            }
        }
    }
    grid_barrier(bar, nb);
    if (MODE == HIER_PDA) {
        for (int k = 1; k <= top; ++k) {
            const HLevel& L = h.lv[k];
            const double zw = pow(h.alpha, -(h.beta + (double)k));
            float* mu = const_cast<float*>(L.mu);
            for (int64_t p = gtid; p < L.M; p += gstride) {
                const int f = (int)(L.keys[p] >> 56);
                const float den = L.buf[p];
                mu[p] = (k < h.frameLevels[f] && den > 0.f) ? (float)(zw * (double)L.count[p] / (double)den) : 0.f;
            }
        }
        return;
    }
    // ---- project kc−1 → 1 (grid-wide)
    for (int k = kc - 1; k >= 1; --k) {
        project_level(k, 0, h.lv[k].M, gtid, gstride);
        grid_barrier(bar, nb);
    }
    if (!do_level0) return;
    // ---- level 0
    const float* acc1 = h.lv[1].buf;
    const int64_t M1 = h.lv[1].M;
    const int* parent0 = h.lv[0].parent;
    if (MODE == HIER_INIT) {
        const int K = C - 1;
        for (int64_t v = gtid; v < a.M; v += gstride) {
            const int pa = parent0[v];
            const float den = in0[(size_t)K * a.M + v] + acc1[(size_t)K * M1 + pa];
            for (int k = 0; k < K; ++k) {
                const float num = in0[(size_t)k * a.M + v] + acc1[(size_t)k * M1 + pa];
                out0[(size_t)k * a.M + v] = (den > 0.f) ? num / den : 0.f;
            }
        }
        return;
    }
    if (MODE == HIER_PLAIN) {
        for (int64_t v = gtid; v < a.M; v += gstride) {
            const int pa = parent0[v];
            const float m0 = a.mu0[v];
            for (int k = 0; k < a.K; ++k) {
                const float s = (m0 > 0.f) ? m0 * in0[(size_t)k * a.M + v] + acc1[(size_t)k * M1 + pa] : 0.f;
                out0[(size_t)k * a.M + v] = s;
            }
        }
        return;
    }
    // HIER_PCG: per-frame blocks
    const int f = blockIdx.x / bpf, j = blockIdx.x % bpf;
    const int v0 = a.frameOff[f], v1 = a.frameOff[f + 1];
    const int stride = bpf * blockDim.x;
    for (int k = 0; k < a.K; ++k) {
        const int fk = f * a.K + k;
        double rho = 0.0, rr = 0.0;
        if (first || a.sc_.active[fk]) {
            const size_t off = (size_t)k * a.M;
            const float* ac = acc1 + (size_t)k * M1;
            for (int v0u = v0 + j * blockDim.x + threadIdx.x; v0u < v1; v0u += 4 * stride) {
                float rv[4], mv[4], up[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int v = v0u + u * stride;
                    if (v < v1) {
                        rv[u] = a.r[off + v];
                        mv[u] = a.mu0[v];
                        up[u] = ac[parent0[v]];
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int v = v0u + u * stride;
                    if (v >= v1) continue;
                    const float sval = (mv[u] > 0.f) ? mv[u] * rv[u] + up[u] : 0.f;
                    a.s[off + v] = sval;
                    rho += (double)rv[u] * (double)sval;
                    rr += (double)rv[u] * (double)rv[u];
                }
            }
        }
        rho = block_sum(rho, shd);
        rr = block_sum(rr, shd);
        if (threadIdx.x == 0) {
            double* pp = a.partial + ((size_t)f * bpf + j) * 2 * a.K + 2 * k;
            pp[0] = rho;
            pp[1] = rr;
        }
    }
    if (last_block_of_frame(a.counters + f, bpf, &sflag)) {
        VecArgs b = a;
        b.BPF = bpf;
        finish_rho(b, f, first != 0, shd);
    }
}


// Level 0 → 1 lift of P as a full-occupancy kernel: thread per level-1 parent,
// children read in canonical child order (deterministic), 4 child loads in flight.
__global__ void __launch_bounds__(256) k_lift01(const float* __restrict__ in0, int64_t M0, const int* __restrict__ cs,
                                                const int* __restrict__ cl, int64_t M1, int C, float* __restrict__ out1) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < M1; p += (int64_t)gridDim.x * blockDim.x) {
        const int q0 = cs[p], q1 = cs[p + 1];
        for (int c = 0; c < C; ++c) {
            const float* src = in0 + (size_t)c * M0;
            float acc = 0.f;
            int q = q0;
            for (; q + 4 <= q1; q += 4) {
                const int i0 = cl[q], i1 = cl[q + 1], i2 = cl[q + 2], i3 = cl[q + 3];
                const float v0 = src[i0], v1 = src[i1], v2 = src[i2], v3 = src[i3];
                acc += v0;
                acc += v1;
                acc += v2;
                acc += v3;
            }
            for (; q < q1; ++q) acc += src[cl[q]];
            out1[(size_t)c * M1 + p] = acc;
        }
    }
}
}  // namespace fbs
