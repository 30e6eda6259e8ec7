// grid_kernels.cuh — simplified bilateral grid on sm_100a.
//
// Canonical vertex order is ascending packed key frame‖by‖bx‖bl‖bu‖bv (reading #3).  The
// (frame, by, bx) digits of a pixel's key follow from its position, so the vertices of one
// σxy×σxy cell are contiguous and cells appear in raster order: the grid is built by a
// cell-local sort of the 24-bit (bl, bu, bv) codes (one warp per cell) plus a single-pass
// decoupled look-back scan of per-cell unique counts for the global vertex ids — no global
// sort of N keys is needed.
#pragma once
#include "fbs_common.cuh"

namespace fbs {

// ---------------------------------------------------------------- axis bins (reading #2)
// start[b] = first coordinate i with ⌊i/σ⌋ = b; start[nb] = len.  σ ≥ 1, so bins are dense.
__global__ void k_axis_bins(int len, double sigma, int nb, int* __restrict__ start) {
    pdl_entry();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) {
        const int b = (int)floor((double)i / sigma);
        const int bp = (i == 0) ? -1 : (int)floor((double)(i - 1) / sigma);
        if (b != bp) start[b] = i;
        if (i == len - 1) start[nb] = len;
    }
}

struct CellGeom {
    int F, H, W, ncx, ncy;
    const int* colStart;
    const int* rowStart;
};

// ---------------------------------------------------------------- warp bitonic sort, 64 keys
// element e = j*32 + lane (a0: j = 0, a1: j = 1); ascending.
__device__ __forceinline__ void warp_bitonic64(uint32_t& a0, uint32_t& a1, int lane) {
#pragma unroll
    for (int k = 2; k <= 64; k <<= 1) {
#pragma unroll
        for (int s = k >> 1; s > 0; s >>= 1) {
            if (s == 32) {
                const bool asc = (lane & k) == 0;
                const uint32_t lo = min(a0, a1), hi = max(a0, a1);
                a0 = asc ? lo : hi;
                a1 = asc ? hi : lo;
            } else {
                const uint32_t p0 = __shfl_xor_sync(0xffffffffu, a0, s);
                const uint32_t p1 = __shfl_xor_sync(0xffffffffu, a1, s);
                const bool lower = (lane & s) == 0;
                const bool asc0 = (lane & k) == 0;
                const bool asc1 = ((lane + 32) & k) == 0;
                a0 = (lower == asc0) ? min(a0, p0) : max(a0, p0);
                a1 = (lower == asc1) ? min(a1, p1) : max(a1, p1);
            }
        }
    }
}

// Bin tables: lut[i] = ⌊i / d⌋ for every integer numerator i ∈ [0, 65536), one IEEE fp64 division
// each (reading #2), d = 256σ.  Yn, Un, Vn are integers < 65536, so a table lookup reproduces the
// fp64 division exactly while keeping the per-pixel path free of fp64 divides.
__global__ void k_bin_lut(double d, uint8_t* __restrict__ lut) {
    pdl_entry();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < 65536) lut[i] = (uint8_t)min(255.0, floor((double)i / d));
}

// (bl, bu, bv) code of one pixel: reading #1 integer YUV numerators, reading #2 bins (tables).
__device__ __forceinline__ uint32_t luv_code(const uint8_t* __restrict__ px, const uint8_t* __restrict__ lutL,
                                            const uint8_t* __restrict__ lutUV) {
    const int R = px[0], G = px[1], B = px[2];
    const int Yn = 77 * R + 150 * G + 29 * B;
    const int Un = -43 * R - 85 * G + 128 * B + 32768;
    const int Vn = 128 * R - 107 * G - 21 * B + 32768;
    const uint32_t bl = __ldg(lutL + Yn), bu = __ldg(lutUV + Un), bv = __ldg(lutUV + Vn);
    return (bl << 16) | (bu << 8) | bv;
}

__device__ __forceinline__ void cell_of(const CellGeom& g, int64_t c, int& f, int& cy, int& cx) {
    // 32-bit arithmetic (cell counts < 2^31; a 64-bit division is a ~70-instruction sequence)
    const unsigned per = (unsigned)g.ncx * (unsigned)g.ncy, cu = (unsigned)c;
    f = (int)(cu / per);
    const unsigned r = cu - (unsigned)f * per;
    cy = (int)(r / (unsigned)g.ncx);
    cx = (int)(r - (unsigned)cy * (unsigned)g.ncx);
}

// ---------------------------------------------------------------- level-0 grid build
// Three passes (count → scan → write), so no pass waits on a serial inter-block chain:
//   k_grid_sort   one warp per σxy cell (≤ 64 px): 24-bit (l,u,v) codes of the pixels, a
//                 64-element warp bitonic sort of (code‖pixel), run heads → the cell's unique
//                 count, its head bitmask and its sorted pixel permutation (1 B/px).
//   k_scan_excl   exclusive scan of the per-cell counts → cellOff (global canonical vertex ids).
//   k_grid_write  per cell: vid[p] = cellOff + rank of p's run, keys/m of every run head.
// Outputs: keys[v], m[v] (= S1), vid[p], cellOff[c] (first vertex of each cell), perm.
__global__ void __launch_bounds__(256) k_grid_sort(
    const uint8_t* __restrict__ rgb, CellGeom g, const uint8_t* __restrict__ lutL,
    const uint8_t* __restrict__ lutUV, int64_t ncells, int* __restrict__ cnt,
    unsigned long long* __restrict__ heads, uint8_t* __restrict__ perm, int* __restrict__ err) {
    pdl_entry();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t c = (int64_t)blockIdx.x * kCellsPerBlock + warp; c < ncells;
         c += (int64_t)gridDim.x * kCellsPerBlock) {
        int f, cy, cx;
        cell_of(g, c, f, cy, cx);
        const int x0 = g.colStart[cx], y0 = g.rowStart[cy];
        const int w = g.colStart[cx + 1] - x0;
        const int h = g.rowStart[cy + 1] - y0;
        int npx = w * h;
        if (npx > kCellMaxPx) {  // host validated σxy ≤ 8; keep the kernel safe anyway
            if (lane == 0) atomicOr(err, 1);
            npx = kCellMaxPx;
        }
        const uint8_t* base = rgb + (size_t)f * g.H * g.W * 3;
        const float rw = 1.f / (float)w;  // (i + ½)/w is ≥ 1/128 from an integer: exact row
        uint32_t a0 = 0xffffffffu, a1 = 0xffffffffu;
        if (lane < npx) {
            const int iy = (int)(((float)lane + 0.5f) * rw);
            const int px = x0 + lane - iy * w, py = y0 + iy;
            a0 = (luv_code(base + ((size_t)py * g.W + px) * 3, lutL, lutUV) << 6) | (uint32_t)(iy << 3 | (lane - iy * w));
        }
        if (lane + 32 < npx) {
            const int i = lane + 32;
            const int iy = (int)(((float)i + 0.5f) * rw);
            const int px = x0 + i - iy * w, py = y0 + iy;
            a1 = (luv_code(base + ((size_t)py * g.W + px) * 3, lutL, lutUV) << 6) | (uint32_t)(iy << 3 | (i - iy * w));
        }
        warp_bitonic64(a0, a1, lane);
        // run heads in sorted order (same code ⇒ same vertex)
        const uint32_t up0 = __shfl_up_sync(0xffffffffu, a0, 1);
        const uint32_t up1 = __shfl_up_sync(0xffffffffu, a1, 1);
        const uint32_t last0 = __shfl_sync(0xffffffffu, a0, 31);
        const uint32_t prev1 = lane ? up1 : last0;
        const bool v0 = a0 != 0xffffffffu, v1 = a1 != 0xffffffffu;
        const bool h0 = v0 && (lane == 0 || (up0 >> 6) != (a0 >> 6));
        const bool h1 = v1 && ((prev1 >> 6) != (a1 >> 6));
        const unsigned hb0 = __ballot_sync(0xffffffffu, h0);
        const unsigned hb1 = __ballot_sync(0xffffffffu, h1);
        // sorted position → the pixel's (row, column) in the cell as row·8 + column (w, h ≤ 8): the
        // same order as the row-major pixel index for equal codes, and no division to decode
        if (v0) perm[(size_t)c * kCellMaxPx + lane] = (uint8_t)(a0 & 63u);
        if (v1) perm[(size_t)c * kCellMaxPx + lane + 32] = (uint8_t)(a1 & 63u);
        if (lane == 0) {
            cnt[c] = __popc(hb0) + __popc(hb1);
            heads[c] = (unsigned long long)hb0 | ((unsigned long long)hb1 << 32);
        }
    }
}

// Exclusive scan of n ints → out[0..n] (out[n] = total), one pass: tiles of kScanBlock·kScanItems
// values with a warp-parallel decoupled look-back (few tiles ⇒ a short chain).  frameOff (if not
// null): frameOff[i / per] = out[i] for i a multiple of per (per-frame offsets of cell-ordered
// counts).
constexpr int kScanBlock = 256, kScanItems = 16;
__global__ void __launch_bounds__(kScanBlock) k_scan_excl(const int* __restrict__ in, int64_t n, int* __restrict__ out,
                                                        unsigned* __restrict__ tile_counter,
                                                        unsigned long long* __restrict__ tile_state, int64_t per,
                                                        int* __restrict__ frameOff) {
    pdl_entry();
    __shared__ unsigned s_tile;
    __shared__ int s_warp[kScanBlock / 32];
    __shared__ unsigned s_excl;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const unsigned tile = s_tile;
    const int64_t base = (int64_t)tile * kScanBlock * kScanItems + (int64_t)threadIdx.x * kScanItems;
    int v[kScanItems];
    int sum = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        v[i] = (base + i < n) ? in[base + i] : 0;
        sum += v[i];
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[w] = incl;
    __syncthreads();
    int wex = 0, agg = 0;
    for (int i = 0; i < kScanBlock / 32; ++i) {
        if (i < w) wex += s_warp[i];
        agg += s_warp[i];
    }
    if (w == 0) {
        const unsigned long long ex = lookback_warp(tile_state, tile, lb_pack((unsigned)agg, 0u));
        if (lane == 0) s_excl = lb_first(ex);
    }
    __syncthreads();
    int run = (int)s_excl + wex + incl - sum;
    int64_t fq = frameOff ? base / per : 0, fr = frameOff ? base - fq * per : 0;  // base = fq·per + fr
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        if (base + i < n) {
            out[base + i] = run;
            if (frameOff && fr == 0) frameOff[fq] = run;
        }
        if (++fr == per) {
            fr = 0;
            ++fq;
        }
        if (base + i == n - 1) {
            out[n] = run + v[i];
            if (frameOff) frameOff[n / per] = run + v[i];
        }
        run += v[i];
    }
    if (n == 0 && tile == 0 && threadIdx.x == 0) {
        out[0] = 0;
        if (frameOff) frameOff[0] = 0;
    }
}

__global__ void __launch_bounds__(256, 8) k_grid_write(
    const uint8_t* __restrict__ rgb, CellGeom g, const uint8_t* __restrict__ lutL,
    const uint8_t* __restrict__ lutUV, int64_t ncells, const int* __restrict__ cellOff,
    const unsigned long long* __restrict__ heads, const uint8_t* __restrict__ perm, uint64_t* __restrict__ keys,
    int* __restrict__ mcount, int* __restrict__ vid) {
    pdl_entry();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int c = blockIdx.x * kCellsPerBlock + warp; c < (int)ncells;  // cells ≤ pixels < 2^31
         c += gridDim.x * kCellsPerBlock) {
        int f, cy, cx;
        cell_of(g, c, f, cy, cx);
        const int x0 = g.colStart[cx], y0 = g.rowStart[cy];
        const int w = g.colStart[cx + 1] - x0;
        const int npx = min(w * (g.rowStart[cy + 1] - y0), kCellMaxPx);
        const unsigned long long H64 = heads[c];
        const unsigned off = (unsigned)cellOff[c];
        const uint64_t khi = ((uint64_t)f << 56) | ((uint64_t)cy << 40) | ((uint64_t)cx << 24);
        const uint8_t* base = rgb + (size_t)f * g.H * g.W * 3;
        int* vbase = vid + (size_t)f * g.H * g.W;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int e = lane + 32 * j;
            if (e >= npx) continue;
            const int i = perm[(size_t)c * kCellMaxPx + e];  // row·8 + column
            const int px = x0 + (i & 7), py = y0 + (i >> 3);
            const unsigned long long upto = (e == 63) ? ~0ull : ((2ull << e) - 1ull);
            const unsigned v = off + (unsigned)__popcll(H64 & upto) - 1u;
            vbase[(size_t)py * g.W + px] = (int)v;
            if ((H64 >> e) & 1ull) {
                const unsigned long long rest = H64 & ~upto;
                const int nxt = rest ? (__ffsll((long long)rest) - 1) : npx;
                keys[v] = khi | (uint64_t)luv_code(base + ((size_t)py * g.W + px) * 3, lutL, lutUV);
                mcount[v] = nxt - e;
            }
        }
    }
}

// ---------------------------------------------------------------- neighbours (B̄ structure)
// position of code q in a sorted shared-memory segment padded to 64 entries with 0xFFFFFFFF
// (codes are 24-bit, so the padding sorts last and never matches): 6 fixed, branch-free steps
__device__ __forceinline__ int find_s(const uint32_t* a, uint32_t q) {
    int pos = 0;
#pragma unroll
    for (int step = 32; step > 0; step >>= 1)
        if (a[pos + step - 1] < q) pos += step;
    return (a[pos] == q) ? pos : -1;
}

// One warp per cell: stage the 24-bit codes of the cell and of its x∓ / y∓ neighbour cells in
// shared memory, then each vertex finds its 10 ±1 neighbours (reading #4): v± are adjacent in the
// sorted cell, the other 8 are binary searches.
__global__ void __launch_bounds__(256) k_grid_neighbours(
    const uint64_t* __restrict__ keys, const int* __restrict__ cellOff, int ncx, int ncy,
    int64_t ncells, int4* __restrict__ nbr, int* __restrict__ err) {
    pdl_entry();
    __shared__ uint32_t sc[kCellsPerBlock][5][kCellMaxPx + 1];  // + 1: sc[i + 1] of the last entry
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // 32-bit cell arithmetic (cells ≤ pixels < 2^31); codes are the low words of the keys
    const uint32_t* keys32 = reinterpret_cast<const uint32_t*>(keys);
    const int nc = (int)ncells;
    const unsigned per = (unsigned)ncx * (unsigned)ncy;
    int bad = 0;
    for (int c = blockIdx.x * kCellsPerBlock + warp; c < nc; c += gridDim.x * kCellsPerBlock) {
        const unsigned r = (unsigned)c % per;
        const int cy = (int)(r / (unsigned)ncx), cx = (int)(r - (unsigned)cy * (unsigned)ncx);
        int st[5], ln[5];
        const int cc[5] = {c, c - 1, c + 1, c - ncx, c + ncx};
        const bool ok[5] = {true, cx > 0, cx < ncx - 1, cy > 0, cy < ncy - 1};
#pragma unroll
        for (int s = 0; s < 5; ++s) {
            st[s] = ok[s] ? cellOff[cc[s]] : 0;
            ln[s] = ok[s] ? cellOff[cc[s] + 1] - st[s] : 0;
            if (ln[s] > kCellMaxPx) {
                if (lane == 0) atomicOr(err, 2);
                ln[s] = kCellMaxPx;
            }
#pragma unroll
            for (int h = 0; h < kCellMaxPx / 32; ++h) {
                const int i = lane + 32 * h;
                sc[warp][s][i] = (i < ln[s]) ? (__ldg(keys32 + 2 * (size_t)(st[s] + i)) & 0xffffffu) : 0xffffffffu;
            }
        }
        if (lane == 0) sc[warp][0][kCellMaxPx] = 0xffffffffu;
        __syncwarp();
        for (int i = lane; i < ln[0]; i += 32) {
            const uint32_t q = sc[warp][0][i];
            const int v = st[0] + i;
            const uint32_t l = (q >> 16) & 255u, u = (q >> 8) & 255u, vv = q & 255u;
            // slot order x−, x+, l−, l+, u−, u+, v−, v+, y−, y+.  v± (the least significant field)
            // are the adjacent entries of the cell's sorted codes when present; the rest are
            // searched in the staged segment of their cell (x∓: cells c∓1, y∓: c∓ncx, else c).
            int offs[10];
            const int seg[6] = {1, 2, 0, 0, 0, 0};
            const uint32_t tq[6] = {q, q, q - (1u << 16), q + (1u << 16), q - (1u << 8), q + (1u << 8)};
            const bool in[6] = {true, true, l > 0, l < 255, u > 0, u < 255};
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                const int s = seg[k];
                const int j = in[k] ? find_s(sc[warp][s], tq[k]) : -1;
                offs[k] = (j >= 0) ? st[s] + j - v : 0;
            }
            offs[6] = (vv > 0 && i > 0 && sc[warp][0][i - 1] == q - 1u) ? -1 : 0;
            offs[7] = (vv < 255 && sc[warp][0][i + 1] == q + 1u) ? 1 : 0;  // i + 1 ≤ 64: padded
#pragma unroll
            for (int k = 8; k < 10; ++k) {
                const int s = k - 5;
                const int j = find_s(sc[warp][s], q);
                offs[k] = (j >= 0) ? st[s] + j - v : 0;
            }
            unsigned bx = 0, by = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int o = offs[k];
                bad |= (o < -127 || o > 127);
                const unsigned b = (unsigned)(o & 0xff);
                if (k < 4) bx |= b << (8 * k); else by |= b << (8 * (k - 4));
            }
            nbr[v] = make_int4((int)bx, (int)by, offs[8], offs[9]);
        }
        __syncwarp();
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(err, 4);
}

// ---------------------------------------------------------------- Alg. 1 bistochastization
// n ← sqrt((n ∘ m) / (B̄ n)),  B̄ n = 2D n_v + Σ_{u∈N(v)} n_u, fp32.
// Persistent blocks take chunks of kBsChunk consecutive vertices through a two-stage bulk-copy
// pipeline: while a chunk is computed, the TMA engine copies the next chunk's neighbour structure,
// m and the n window [c0 − 128, c0 + chunk + 128) into shared memory.  The 8 near neighbours
// (|offset| ≤ 127 by construction) are read from the window; only y∓ are global gathers.
// Vertex arrays carry kVecPad slack, so whole 16-byte-multiple copies never leave allocations.
constexpr int kBsChunk = 1024;
constexpr int kBsThreads = 512;
constexpr int kBsWin = kBsChunk + 256;
struct BsStage {
    int4 nb[kBsChunk];
    int m[kBsChunk];
    float n[kBsWin];
};
constexpr size_t kBsSmem = 2 * sizeof(BsStage) + 64;

__global__ void __launch_bounds__(kBsThreads) k_bistoch(const int4* __restrict__ nbr,
                                                 const int* __restrict__ m,
                                                 const float* __restrict__ nin,
                                                 float* __restrict__ nout, const int* __restrict__ frameOff, int F,
                                                 int f0, int f1, int first, float bdiag,
                                                 unsigned* __restrict__ chunkCtr) {
    // The frame offsets were written before the (serialised) launch of k_grid_neighbours that
    // precedes every k_bistoch of a build, so they are complete when any k_bistoch block starts:
    // they are read before waiting on the previous iteration (the first bulk copies go out as soon
    // as the wait returns).
    const int M = frameOff[F], vlo = frameOff[f0], vhi = frameOff[f1];
    pdl_wait();
    extern __shared__ __align__(128) unsigned char bs_smem[];
    BsStage* st = reinterpret_cast<BsStage*>(bs_smem);
    uint64_t* bar = reinterpret_cast<uint64_t*>(bs_smem + 2 * sizeof(BsStage));
    // vertices [vlo, vhi) = frames [f0, f1) (device counts): the chunks covering them; a chunk
    // shared with a neighbouring range only writes its own vertices (no neighbour crosses a frame)
    const int cBeg = vlo / kBsChunk, nChunks = (vhi + kBsChunk - 1) / kBsChunk;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto issue = [&](int slot, int ci) {  // thread 0
        const int c0 = ci * kBsChunk;
        const int n = min(kBsChunk, M - c0);
        const int n4 = (n + 3) & ~3;
        const int w0 = max(c0 - 128, 0);                 // 16-byte aligned (c0 is a multiple of 1024)
        const int w1 = min(c0 + kBsChunk + 128, (M + 3) & ~3);
        const uint32_t bytes = (uint32_t)(n * 16 + n4 * 4 + (first ? 0 : (w1 - w0) * 4));
        mbar_expect_tx(&bar[slot], bytes);
#ifndef FBS_BS_NO_HINT
        // the neighbour structure (16 of 28 B per vertex) streams evict-first; m and n, re-read by
        // every iteration, are kept (evict-last): 30.2 -> 28.5 µs per launch, 5.14 -> 5.10 ms per step
        bulk_g2s_hint(st[slot].nb, nbr + c0, n * 16, &bar[slot], l2_policy_evict_first());
        bulk_g2s_hint(st[slot].m, m + c0, n4 * 4, &bar[slot], l2_policy_evict_last());
        if (!first)
            bulk_g2s_hint(st[slot].n + (w0 - (c0 - 128)), nin + w0, (w1 - w0) * 4, &bar[slot], l2_policy_evict_last());
#else
        bulk_g2s(st[slot].nb, nbr + c0, n * 16, &bar[slot]);
        bulk_g2s(st[slot].m, m + c0, n4 * 4, &bar[slot]);
        if (!first) bulk_g2s(st[slot].n + (w0 - (c0 - 128)), nin + w0, (w1 - w0) * 4, &bar[slot]);
#endif
    };
    // chunkCtr (dynamic scheduling): blocks take chunks from a per-launch counter, so a block that
    // starts late (SM slots held by another kernel) takes fewer chunks instead of delaying the
    // launch (28.5 → 26.0 µs per launch in the bench step); each slot's chunk id travels with its
    // stage (sci), and a slot with no chunk left completes its barrier with no bytes (sci = −1)
    volatile int* sci = reinterpret_cast<int*>(bs_smem + 2 * sizeof(BsStage) + 16);
    auto take = [&](int slot, int guess) {  // thread 0: the slot's chunk, issued (or −1)
        const int cj = chunkCtr ? cBeg + (int)atomicAdd(chunkCtr, 1u) : guess;
        sci[slot] = (cj < nChunks) ? cj : -1;
        if (cj < nChunks) issue(slot, cj);
        else mbar_expect_tx(&bar[slot], 0);
    };
    if (threadIdx.x == 0) {
        take(0, cBeg + blockIdx.x);
        take(1, cBeg + blockIdx.x + gridDim.x);
    }
    for (int it = 0;; ++it) {
        const int slot = it & 1;
        mbar_wait(&bar[slot], (it >> 1) & 1);
        const int ci = sci[slot];
        if (ci < 0) break;
        const BsStage& S = st[slot];
        const int c0 = ci * kBsChunk;
        float ny[kBsChunk / kBsThreads][2];
#pragma unroll
        for (int u = 0; u < kBsChunk / kBsThreads; ++u) {
            const int l = threadIdx.x + kBsThreads * u, v = c0 + l;
            const int4 nb = S.nb[l];
            ny[u][0] = (!first && v < M && nb.z) ? __ldg(nin + v + nb.z) : 0.f;
            ny[u][1] = (!first && v < M && nb.w) ? __ldg(nin + v + nb.w) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < kBsChunk / kBsThreads; ++u) {
            const int l = threadIdx.x + kBsThreads * u, v = c0 + l;
            if (v < vlo || v >= vhi) continue;
            const int4 nb = S.nb[l];
            float nv, bn;
            if (first) {
                int deg = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) deg += near_off(nb, i) != 0;
                deg += (nb.z != 0) + (nb.w != 0);
                nv = 1.f;
                bn = bdiag + (float)deg;
            } else {
                const int lv = l + 128;
                nv = S.n[lv];
                float sn = 0.f;  // Σ_{u ∈ N(v)} n_u in the fixed slot order of nbr_sum
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int o = near_off(nb, i);
                    if (o) sn += S.n[lv + o];
                }
                if (nb.z) sn += ny[u][0];
                if (nb.w) sn += ny[u][1];
                bn = bdiag * nv + sn;
            }
            nout[v] = sqrtf(nv * (float)S.m[l] / bn);
        }
        __syncthreads();  // stage `slot` fully consumed (and sci[slot] read by every thread)
        if (threadIdx.x == 0) take(slot, ci + 2 * (int)gridDim.x);
    }
}

// max|n∘B̄n − m| and max m (order-independent max ⇒ deterministic), reporting only.
__global__ void k_bistoch_residual(const int4* __restrict__ nbr,
                                   const int* __restrict__ m, const float* __restrict__ n, int M,
                                   unsigned* __restrict__ out2, float bdiag) {
    pdl_entry();
    float e = 0.f, mm = 0.f;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < M; v += gridDim.x * blockDim.x) {
        const float bn = bdiag * n[v] + nbr_sum(n, v, nbr[v]);
        e = fmaxf(e, fabsf(n[v] * bn - (float)m[v]));
        mm = fmaxf(mm, (float)m[v]);
    }
    for (int o = 16; o; o >>= 1) {
        e = fmaxf(e, __shfl_xor_sync(0xffffffffu, e, o));
        mm = fmaxf(mm, __shfl_xor_sync(0xffffffffu, mm, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(out2, __float_as_uint(e));
        atomicMax(out2 + 1, __float_as_uint(mm));
    }
}

// ---------------------------------------------------------------- exports
__global__ void k_export_nbr(const int4* __restrict__ nbr, int M,
                             int* __restrict__ nbr10) {
    pdl_entry();
    // export slot order (x−,x+,y−,y+,l−,l+,u−,u+,v−,v+); internal near order (x−,x+,l−,l+,u−,u+,v−,v+)
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < M; v += gridDim.x * blockDim.x) {
        const int4 q4 = nbr[v];
        int* o = nbr10 + (size_t)v * 10;
        int nb[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int d = near_off(q4, i);
            nb[i] = d ? v + d : -1;
        }
        o[0] = nb[0];
        o[1] = nb[1];
        o[2] = q4.z ? v + q4.z : -1;
        o[3] = q4.w ? v + q4.w : -1;
        o[4] = nb[2];
        o[5] = nb[3];
        o[6] = nb[4];
        o[7] = nb[5];
        o[8] = nb[6];
        o[9] = nb[7];
    }
}

}  // namespace fbs
