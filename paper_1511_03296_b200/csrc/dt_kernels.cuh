// dt_kernels.cuh — domain-transform recursive-filter post-processing (
// Gastal & Oliveira 2011's RF variant as restated in reading #28).
//
// Each pass is a first-order recursion along a line, J[n] = w[n] J[n−1] + (1 − w[n]) I[n]
// (then the same backwards), i.e. a composition of affine maps.  One warp per line: the line is
// staged in shared memory, lane l composes the maps of its contiguous chunk, a warp scan
// composes the chunk maps, and each lane re-runs its chunk from its incoming value — 2·L/32 + 5
// dependent steps instead of 2·L.  Vertical passes run the same kernel on a tiled transpose.
#pragma once
#include "fbs_common.cuh"

namespace fbs {

// d_x = 1 + ratio Σ_c |I_c(x) − I_c(x−1)| (1 at x = 0), d_y likewise; [F][H][W].
// Grid (⌈W/blockDim⌉, ≤ 65535): rows strided over blockIdx.y, no per-pixel index divisions.
__global__ void k_dt_dist(const uint8_t* __restrict__ rgb, int F, int H, int W, float ratio, float* __restrict__ Dx,
                          float* __restrict__ Dy) {
    pdl_entry();
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= W) return;
    for (int row = blockIdx.y; row < F * H; row += gridDim.y) {  // row = f·H + y
        const int y = row % H;
        const int64_t p = (int64_t)row * W + x;
        const uint8_t* c = rgb + 3 * p;
        float dx = 0.f, dy = 0.f;
        if (x > 0) {
            const uint8_t* l = c - 3;
            dx = fabsf((float)c[0] - l[0]) + fabsf((float)c[1] - l[1]) + fabsf((float)c[2] - l[2]);
        }
        if (y > 0) {
            const uint8_t* u = c - 3 * (int64_t)W;
            dy = fabsf((float)c[0] - u[0]) + fabsf((float)c[1] - u[1]) + fabsf((float)c[2] - u[2]);
        }
        Dx[p] = 1.f + ratio * dx;
        Dy[p] = 1.f + ratio * dy;
    }
}

// The same for W % 4 = 0, four pixels per thread: the 12 bytes of the 4 pixels (and the byte
// triple before them) as 32-bit words, the row above likewise, two 16-byte stores.
__global__ void k_dt_dist4(const uint8_t* __restrict__ rgb, int F, int H, int W, float ratio, float* __restrict__ Dx,
                           float* __restrict__ Dy) {
    pdl_entry();
    const int W4 = W >> 2;
    const int x4 = blockIdx.x * blockDim.x + threadIdx.x;
    if (x4 >= W4) return;
    auto bytes = [](uint32_t w, int i) { return (float)((w >> (8 * i)) & 255u); };
    for (int row = blockIdx.y; row < F * H; row += gridDim.y) {  // row = f·H + y
        const int y = row % H;
        const uint32_t* cw = reinterpret_cast<const uint32_t*>(rgb + ((size_t)row * W + 4 * x4) * 3);
        uint32_t c[4], u[3], pw = 0;  // c[0..2]: the 4 pixels; pw: the word ending with pixel x − 1
        c[0] = __ldg(cw);
        c[1] = __ldg(cw + 1);
        c[2] = __ldg(cw + 2);
        if (x4 > 0) pw = __ldg(cw - 1);
        if (y > 0) {
            const uint32_t* uw = cw - (size_t)W * 3 / 4;  // W % 4 = 0: the row above is word-aligned
            u[0] = __ldg(uw);
            u[1] = __ldg(uw + 1);
            u[2] = __ldg(uw + 2);
        }
        (void)c[3];
        float px[5][3];  // pixels x − 1 … x + 3 (channel bytes in memory order)
        px[0][0] = bytes(pw, 1); px[0][1] = bytes(pw, 2); px[0][2] = bytes(pw, 3);
#pragma unroll
        for (int q = 0; q < 12; ++q) px[1 + q / 3][q % 3] = bytes(c[q / 4], q % 4);
        float dx[4], dy[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float d = fabsf(px[i + 1][0] - px[i][0]) + fabsf(px[i + 1][1] - px[i][1]) + fabsf(px[i + 1][2] - px[i][2]);
            dx[i] = 1.f + ratio * ((x4 > 0 || i > 0) ? d : 0.f);
            float e = 0.f;
            if (y > 0) {
                const int q0 = 3 * i;
                e = fabsf(px[i + 1][0] - bytes(u[q0 / 4], q0 % 4)) + fabsf(px[i + 1][1] - bytes(u[(q0 + 1) / 4], (q0 + 1) % 4)) +
                    fabsf(px[i + 1][2] - bytes(u[(q0 + 2) / 4], (q0 + 2) % 4));
            }
            dy[i] = 1.f + ratio * e;
        }
        const size_t p4 = (size_t)row * W4 + x4;
        reinterpret_cast<float4*>(Dx)[p4] = make_float4(dx[0], dx[1], dx[2], dx[3]);
        reinterpret_cast<float4*>(Dy)[p4] = make_float4(dy[0], dy[1], dy[2], dy[3]);
    }
}

// Transpose of P planes [H][W] → [W][H] through 32×32 shared-memory tiles (coalesced both ways);
// block (32, 8), grid (⌈W/32⌉, ⌈H/32⌉, P).  The column passes run as row passes on the transpose.
__global__ void k_dt_transpose(const float* __restrict__ in, float* __restrict__ out, int H, int W) {
    pdl_entry();
    __shared__ float tile[32][33];
    const size_t plane = (size_t)blockIdx.z * H * W;
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
    for (int j = threadIdx.y; j < 32; j += 8) {
        const int y = y0 + j, x = x0 + threadIdx.x;
        if (y < H && x < W) tile[j][threadIdx.x] = in[plane + (size_t)y * W + x];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += 8) {
        const int x = x0 + j, y = y0 + threadIdx.x;  // out[x][y]
        if (x < W && y < H) out[plane + (size_t)x * H + y] = tile[threadIdx.x][j];
    }
}

constexpr int kDtB = 8;  // loads issued together before their dependent steps

// composition of affine maps J ↦ A J + B: (later ∘ earlier)
__device__ __forceinline__ float2 amap_compose(float2 later, float2 earlier) {
    return make_float2(later.x * earlier.x, later.x * earlier.y + later.y);
}

// Row pass: one causal + anticausal pass along every row of sig [F][K][H][W] (in place),
// w = exp(lna · Dx) with Dx [F][H][W].  One warp per row; the row's values and weights are staged
// in shared memory with coalesced loads (2 · (W + 32) floats per warp: element n at n + n/C, one
// pad slot per lane chunk against bank conflicts).
__global__ void k_dt_rows(float* __restrict__ sig, const float* __restrict__ Dx, int F, int K, int H, int W, float lna) {
    pdl_entry();
    extern __shared__ float dt_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int C = (W + 31) / 32;           // chunk length
    const float invC = 1.f / (float)C;     // ⌊n/C⌋ = ⌊(n + ½)/C⌋ in fp32: exact for n < 2^14·C
    const int lpad = W + 32;
    float* val = dt_smem + (size_t)warp * 2 * lpad;
    float* wgt = val + lpad;
    const int64_t lines = (int64_t)F * K * H;
    for (int64_t r = (int64_t)blockIdx.x * nw + warp; r < lines; r += (int64_t)gridDim.x * nw) {
        const int f = (int)(r / ((int64_t)K * H));
        const int y = (int)(r % H);
        float* line = sig + (size_t)r * W;
        const float* dl = Dx + ((size_t)f * H + y) * W;
        if ((W & 3) == 0) {
            // 16-byte loads (rows start 16-byte aligned when W % 4 = 0): a 1920-pixel line is two
            // rounds of kDtB loads per lane instead of eight — the loads' latency, not bandwidth,
            // bounds a warp's line
            const float4* line4 = reinterpret_cast<const float4*>(line);
            const float4* dl4 = reinterpret_cast<const float4*>(dl);
            const int W4 = W >> 2;
            for (int nb = lane; nb < W4; nb += 32 * kDtB) {
                float4 lv[kDtB], dv[kDtB];
#pragma unroll
                for (int u = 0; u < kDtB; ++u) {
                    const int n4 = nb + 32 * u;
                    lv[u] = (n4 < W4) ? line4[n4] : make_float4(0.f, 0.f, 0.f, 0.f);
                    dv[u] = (n4 < W4) ? __ldg(dl4 + n4) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < kDtB; ++u) {
                    const int n4 = nb + 32 * u;
                    if (n4 < W4) {
                        const float le[4] = {lv[u].x, lv[u].y, lv[u].z, lv[u].w};
                        const float de[4] = {dv[u].x, dv[u].y, dv[u].z, dv[u].w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int n = 4 * n4 + e;
                            const int pn = n + __float2int_rz(((float)n + 0.5f) * invC);
                            val[pn] = le[e];
                            wgt[pn] = (n == 0) ? 0.f : __expf(lna * de[e]);
                        }
                    }
                }
            }
        } else {
            for (int nb = lane; nb < W; nb += 32 * kDtB) {  // kDtB loads of each array in flight
                float lv[kDtB], dv[kDtB];
#pragma unroll
                for (int u = 0; u < kDtB; ++u) {
                    const int n = nb + 32 * u;
                    lv[u] = (n < W) ? line[n] : 0.f;
                    dv[u] = (n < W) ? __ldg(dl + n) : 0.f;
                }
#pragma unroll
                for (int u = 0; u < kDtB; ++u) {
                    const int n = nb + 32 * u;
                    if (n < W) {
                        const int pn = n + __float2int_rz(((float)n + 0.5f) * invC);
                        val[pn] = lv[u];
                        wgt[pn] = (n == 0) ? 0.f : __expf(lna * dv[u]);  // w[0] = 0: the first element keeps its value
                    }
                }
            }
        }
        __syncwarp();
        const int n0 = lane * C, n1 = min(n0 + C, W);
        const int base = lane * (C + 1);  // padded index of n0
        // causal: map_n = (w[n], (1 − w[n]) I[n])
        float2 m = make_float2(1.f, 0.f);
        for (int q = base; q < base + (n1 - n0); ++q) m = amap_compose(make_float2(wgt[q], (1.f - wgt[q]) * val[q]), m);
        float2 incl = m;  // inclusive warp scan (lanes in increasing order)
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const float ax = __shfl_up_sync(0xffffffffu, incl.x, o), ay = __shfl_up_sync(0xffffffffu, incl.y, o);
            if (lane >= o) incl = amap_compose(incl, make_float2(ax, ay));
        }
        float J = __shfl_up_sync(0xffffffffu, incl.y, 1);  // value entering the chunk (maps chain from A = 0)
        for (int q = base; q < base + (n1 - n0); ++q) {
            J = wgt[q] * J + (1.f - wgt[q]) * val[q];
            val[q] = J;
        }
        __syncwarp();
        // anticausal: element n uses w[n+1] (0 for the last element); the padded position of n+1
        // is q+1 inside the chunk and q+2 across the next chunk's pad slot
        auto wnext = [&](int n, int q) { return (n + 1 < W) ? wgt[(n + 1 == n1) ? q + 2 : q + 1] : 0.f; };
        m = make_float2(1.f, 0.f);
        for (int n = n1 - 1, q = base + (n1 - 1 - n0); n >= n0; --n, --q) {
            const float w = wnext(n, q);
            m = amap_compose(make_float2(w, (1.f - w) * val[q]), m);
        }
        incl = m;  // inclusive scan in decreasing lane order
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const float ax = __shfl_down_sync(0xffffffffu, incl.x, o), ay = __shfl_down_sync(0xffffffffu, incl.y, o);
            if (lane + o < 32) incl = amap_compose(incl, make_float2(ax, ay));
        }
        J = __shfl_down_sync(0xffffffffu, incl.y, 1);
        for (int n = n1 - 1, q = base + (n1 - 1 - n0); n >= n0; --n, --q) {
            const float w = wnext(n, q);
            J = w * J + (1.f - w) * val[q];
            val[q] = J;
        }
        __syncwarp();
        for (int n = lane; n < W; n += 32) line[n] = val[n + __float2int_rz(((float)n + 0.5f) * invC)];
        __syncwarp();
    }
}

// Row pass with TWO warps per row (rows of ≥ 256 pixels): warp 2p + h of a block handles half h
// of row p, [h·Wh, min((h+1)·Wh, W)) with Wh a multiple of 4, staged and chunked exactly as in
// k_dt_rows.  The halves exchange one value through shared memory per direction: the causal
// value leaving half 0 (its composed map applied to the row's start, whose weight is 0) and the
// anticausal value leaving half 1.  Half the shared memory per warp and half the serial chunk
// walk of k_dt_rows.  Block: 8 warps = 4 rows; every row of a block runs in step (__syncthreads).
constexpr int kDtB2 = 4;  // 16-byte loads of each array in flight per lane (3 blocks per SM)
__global__ void __launch_bounds__(256, 3) k_dt_rows2(float* __restrict__ sig, const float* __restrict__ Dx, int F, int K, int H, int W,
                           float lna) {
    pdl_entry();
    extern __shared__ float dt_smem[];
    __shared__ float xch[2][4];  // [direction][row of the block]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rb = warp >> 1, h = warp & 1;  // row of the block, half
    const int Wh = ((W + 1) / 2 + 3) & ~3;
    const int a = h * Wh, b = min(a + Wh, W), L = b - a;  // this warp's elements (L ≥ 1 for W ≥ 8)
    const int C = (Wh + 31) / 32;
    const float invC = 1.f / (float)C;
    const int lpad = Wh + 32 + 1;  // + 1: the next half's first weight (anticausal, half 0)
    float* val = dt_smem + (size_t)warp * 2 * lpad;
    float* wgt = val + lpad;
    const int64_t lines = (int64_t)F * K * H;
    for (int64_t r0 = (int64_t)blockIdx.x * 4; r0 < lines; r0 += (int64_t)gridDim.x * 4) {
        const int64_t r = r0 + rb;
        const bool live = r < lines;
        float* line = sig + (size_t)(live ? r : 0) * W;
        const int f = live ? (int)(r / ((int64_t)K * H)) : 0;
        const int y = live ? (int)(r % H) : 0;
        const float* dl = Dx + ((size_t)f * H + y) * W;
        auto pidx = [&](int n) { return n + __float2int_rz(((float)n + 0.5f) * invC); };  // local n
        if (live) {
            const float4* line4 = reinterpret_cast<const float4*>(line + a);
            const float4* dl4 = reinterpret_cast<const float4*>(dl + a);
            const int L4 = (L + 3) >> 2;
            for (int nb = lane; nb < L4; nb += 32 * kDtB2) {
                float4 lv[kDtB2], dv[kDtB2];
#pragma unroll
                for (int u = 0; u < kDtB2; ++u) {
                    const int n4 = nb + 32 * u;
                    lv[u] = (n4 < L4) ? line4[n4] : make_float4(0.f, 0.f, 0.f, 0.f);
                    dv[u] = (n4 < L4) ? __ldg(dl4 + n4) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < kDtB2; ++u) {
                    const int n4 = nb + 32 * u;
                    if (n4 < L4) {
                        const float le[4] = {lv[u].x, lv[u].y, lv[u].z, lv[u].w};
                        const float de[4] = {dv[u].x, dv[u].y, dv[u].z, dv[u].w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int n = 4 * n4 + e;  // local (W % 4 = 0: L % 4 = 0)
                            val[pidx(n)] = le[e];
                            wgt[pidx(n)] = (a + n == 0) ? 0.f : __expf(lna * de[e]);
                        }
                    }
                }
            }
            // w[b] where wnext reads it for half 0's last element (two past its padded index)
            if (h == 0 && lane == 0) wgt[pidx(L - 1) + 2] = (b < W) ? __expf(lna * __ldg(dl + b)) : 0.f;
        }
        __syncwarp();
        const int n0 = min(lane * C, L), n1 = min(n0 + C, L);
        const int base = lane * (C + 1);  // padded index of n0
        // causal: lane chunk maps, warp scan, then the value entering this half
        float2 m = make_float2(1.f, 0.f);
        for (int q = base; q < base + (n1 - n0); ++q) m = amap_compose(make_float2(wgt[q], (1.f - wgt[q]) * val[q]), m);
        float2 incl = m;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const float ax = __shfl_up_sync(0xffffffffu, incl.x, o), ay = __shfl_up_sync(0xffffffffu, incl.y, o);
            if (lane >= o) incl = amap_compose(incl, make_float2(ax, ay));
        }
        if (h == 0 && lane == 31) xch[0][rb] = incl.y;  // half 0 starts at w = 0: its map is (0, J_end)
        __syncthreads();
        const float Jin = (h == 0) ? 0.f : xch[0][rb];
        const float ex = __shfl_up_sync(0xffffffffu, incl.x, 1), ey = __shfl_up_sync(0xffffffffu, incl.y, 1);
        float J = (lane == 0) ? Jin : ex * Jin + ey;
        for (int q = base; q < base + (n1 - n0); ++q) {
            J = wgt[q] * J + (1.f - wgt[q]) * val[q];
            val[q] = J;
        }
        __syncwarp();
        // anticausal: local n uses w[n+1] (the last element of the row 0; half 0's last element
        // the staged first weight of half 1)
        auto wnext = [&](int n, int q) {
            if (a + n + 1 >= W) return 0.f;
            return wgt[(n + 1 == n1) ? q + 2 : q + 1];
        };
        m = make_float2(1.f, 0.f);
        for (int n = n1 - 1, q = base + (n1 - 1 - n0); n >= n0; --n, --q) {
            const float w = wnext(n, q);
            m = amap_compose(make_float2(w, (1.f - w) * val[q]), m);
        }
        incl = m;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const float ax = __shfl_down_sync(0xffffffffu, incl.x, o), ay = __shfl_down_sync(0xffffffffu, incl.y, o);
            if (lane + o < 32) incl = amap_compose(incl, make_float2(ax, ay));
        }
        if (h == 1 && lane == 0) xch[1][rb] = incl.y;  // half 1 ends at w = 0: its map is (0, J_start)
        __syncthreads();
        const float Jin2 = (h == 1) ? 0.f : xch[1][rb];
        const float fx = __shfl_down_sync(0xffffffffu, incl.x, 1), fy = __shfl_down_sync(0xffffffffu, incl.y, 1);
        J = (lane == 31) ? Jin2 : fx * Jin2 + fy;
        for (int n = n1 - 1, q = base + (n1 - 1 - n0); n >= n0; --n, --q) {
            const float w = wnext(n, q);
            J = w * J + (1.f - w) * val[q];
            val[q] = J;
        }
        __syncwarp();
        if (live)
            for (int n = lane; n < L; n += 32) line[a + n] = val[pidx(n)];
        __syncthreads();
    }
}

// Column pass, in place on the row-major sig [F][K][H][W], w = exp(lna · Dy) with Dy [F][H][W]:
// one block per 32 adjacent columns of one (frame, channel) plane; lane = column (coalesced
// 128-byte row segments), warp = a chunk of rows.  Each lane composes its chunk's maps, the
// chunk maps of a column are scanned across warps in shared memory, and the chunk is re-run
// from its incoming value (values re-read from L2).  Rows are processed in batches of kDtB with
// every load of the batch issued before its dependent compose/apply steps.
__global__ void __launch_bounds__(1024) k_dt_cols(float* __restrict__ sig, const float* __restrict__ Dy, int F, int K,
                                                  int H, int W, float lna) {
    pdl_entry();
    __shared__ float2 cm[32][33];  // [warp][lane] chunk maps
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int tilesX = (W + 31) / 32;
    const int64_t planes = (int64_t)F * K;
    const int R = (H + nw - 1) / nw;  // rows per chunk
    for (int64_t b = blockIdx.x; b < planes * tilesX; b += gridDim.x) {
        const int64_t pl = b / tilesX;
        const int x = (int)(b % tilesX) * 32 + lane;
        const int f = (int)(pl / K);
        const bool ok = x < W;
        float* col = sig + (size_t)pl * H * W + (ok ? x : 0);
        const float* dcol = Dy + (size_t)f * H * W + (ok ? x : 0);
        const int y0 = warp * R, y1 = ok ? min(y0 + R, H) : y0;
        float wv[kDtB], iv[kDtB];
        // causal: row y uses w[y] (w = 0 at y = 0)
        float2 m = make_float2(1.f, 0.f);
        for (int yb = y0; yb < y1; yb += kDtB) {
#pragma unroll
            for (int u = 0; u < kDtB; ++u) {
                const int y = yb + u;
                wv[u] = (y < y1 && y > 0) ? __ldg(dcol + (size_t)y * W) : 0.f;
                iv[u] = (y < y1) ? col[(size_t)y * W] : 0.f;
            }
#pragma unroll
            for (int u = 0; u < kDtB; ++u)
                if (yb + u < y1) {
                    const float w = (yb + u > 0) ? __expf(lna * wv[u]) : 0.f;
                    m = amap_compose(make_float2(w, (1.f - w) * iv[u]), m);
                }
        }
        cm[warp][lane] = m;
        __syncthreads();
        float J = 0.f;  // value entering this chunk: maps of the earlier chunks (chained from A = 0)
        for (int q = 0; q < warp; ++q) J = cm[q][lane].x * J + cm[q][lane].y;
        for (int yb = y0; yb < y1; yb += kDtB) {
#pragma unroll
            for (int u = 0; u < kDtB; ++u) {
                const int y = yb + u;
                wv[u] = (y < y1 && y > 0) ? __ldg(dcol + (size_t)y * W) : 0.f;
                iv[u] = (y < y1) ? col[(size_t)y * W] : 0.f;
            }
#pragma unroll
            for (int u = 0; u < kDtB; ++u)
                if (yb + u < y1) {
                    const float w = (yb + u > 0) ? __expf(lna * wv[u]) : 0.f;
                    J = w * J + (1.f - w) * iv[u];
                    col[(size_t)(yb + u) * W] = J;
                }
        }
        __syncthreads();
        // anticausal: row y uses w[y+1]; the last row keeps its value
        m = make_float2(1.f, 0.f);
        for (int yb = y1 - 1; yb >= y0; yb -= kDtB) {
#pragma unroll
            for (int u = 0; u < kDtB; ++u) {
                const int y = yb - u;
                wv[u] = (y >= y0 && y < H - 1) ? __ldg(dcol + (size_t)(y + 1) * W) : 0.f;
                iv[u] = (y >= y0) ? col[(size_t)y * W] : 0.f;
            }
#pragma unroll
            for (int u = 0; u < kDtB; ++u)
                if (yb - u >= y0) {
                    const float w = (yb - u < H - 1) ? __expf(lna * wv[u]) : 0.f;
                    m = amap_compose(make_float2(w, (1.f - w) * iv[u]), m);
                }
        }
        cm[warp][lane] = m;
        __syncthreads();
        J = 0.f;
        for (int q = nw - 1; q > warp; --q) J = cm[q][lane].x * J + cm[q][lane].y;
        for (int yb = y1 - 1; yb >= y0; yb -= kDtB) {
#pragma unroll
            for (int u = 0; u < kDtB; ++u) {
                const int y = yb - u;
                wv[u] = (y >= y0 && y < H - 1) ? __ldg(dcol + (size_t)(y + 1) * W) : 0.f;
                iv[u] = (y >= y0) ? col[(size_t)y * W] : 0.f;
            }
#pragma unroll
            for (int u = 0; u < kDtB; ++u)
                if (yb - u >= y0) {
                    const float w = (yb - u < H - 1) ? __expf(lna * wv[u]) : 0.f;
                    J = w * J + (1.f - w) * iv[u];
                    col[(size_t)(yb - u) * W] = J;
                }
        }
        __syncthreads();
    }
}

// Column pass with the column held in registers (H ≤ kDtColChunks · kDtColRows): one block of
// 64·COLS threads per COLS adjacent columns of one (frame, channel) plane; thread (warp w, lane l)
// owns column l % COLS and chunk w·(32/COLS) + l / COLS of kDtColRows consecutive rows (COLS = 8:
// a warp's loads are four 32-byte row segments, two blocks per SM).  The chunk's values and weights are read once into registers;
// causal and anticausal passes compose the chunk's affine maps, scan the column's chunk maps in
// shared memory (Hillis–Steele, in chunk order) and re-run the chunk from its incoming value;
// the result is stored once: 12 bytes per pixel (sig read and written, Dy read).
constexpr int kDtColRows = 18;  // H ≤ 1152 (registers: 64 per thread at 1024 threads)
constexpr int kDtColChunks = 64;
template <int COLS>  // columns per block: 16 (1024 threads, 64-byte row segments) or 8 (512 threads, 2 blocks/SM)
__global__ void __launch_bounds__(COLS * kDtColChunks, 1024 / (COLS * kDtColChunks)) k_dt_cols_reg(
    float* __restrict__ sig, const float* __restrict__ Dy, int F, int K, int H, int W, float lna) {
    pdl_entry();
    __shared__ float2 cm[kDtColChunks][COLS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int col = lane % COLS, j = warp * (32 / COLS) + lane / COLS;  // chunk index
    const int tilesX = (W + COLS - 1) / COLS;
    const int64_t planes = (int64_t)F * K;
    const int R = (H + kDtColChunks - 1) / kDtColChunks;  // rows per chunk (≤ kDtColRows)
    for (int64_t b = blockIdx.x; b < planes * tilesX; b += gridDim.x) {
        const int64_t pl = b / tilesX;
        const int x = (int)(b % tilesX) * COLS + col;
        const int f = (int)(pl / K);
        const bool ok = x < W;
        float* cs = sig + (size_t)pl * H * W + (ok ? x : 0);
        const float* dc = Dy + (size_t)f * H * W + (ok ? x : 0);
        const int y0 = j * R, y1 = ok ? min(y0 + R, H) : y0;
        float iv[kDtColRows], wv[kDtColRows];
#pragma unroll
        for (int i = 0; i < kDtColRows; ++i) {
            const int y = y0 + i;
            const bool in = i < R && y < y1;
            iv[i] = in ? cs[(size_t)y * W] : 0.f;
            wv[i] = in ? __ldg(dc + (size_t)y * W) : 0.f;
        }
        // the anticausal pass of the chunk's last row needs the next chunk's first weight
        const float dnext = (ok && y1 < H && y1 == y0 + R) ? __ldg(dc + (size_t)y1 * W) : 0.f;
#pragma unroll
        for (int i = 0; i < kDtColRows; ++i) wv[i] = (y0 + i > 0) ? __expf(lna * wv[i]) : 0.f;  // w = 0 at y = 0
        const float wnx = (y1 < H && y1 == y0 + R) ? __expf(lna * dnext) : 0.f;
        // causal: row y uses w[y]
        float2 m = make_float2(1.f, 0.f);
#pragma unroll
        for (int i = 0; i < kDtColRows; ++i)
            if (y0 + i < y1) m = amap_compose(make_float2(wv[i], (1.f - wv[i]) * iv[i]), m);
        cm[j][col] = m;
        __syncthreads();
        // inclusive scan of the column's chunk maps in chunk order (Hillis–Steele, 6 rounds);
        // the incoming value of chunk j is the earlier chunks' composed map applied to 0
#pragma unroll
        for (int r = 1; r < kDtColChunks; r <<= 1) {
            const float2 t = (j >= r) ? amap_compose(cm[j][col], cm[j - r][col]) : cm[j][col];
            __syncthreads();
            cm[j][col] = t;
            __syncthreads();
        }
        float J = (j > 0) ? cm[j - 1][col].y : 0.f;
#pragma unroll
        for (int i = 0; i < kDtColRows; ++i)
            if (y0 + i < y1) {
                J = wv[i] * J + (1.f - wv[i]) * iv[i];
                iv[i] = J;
            }
        __syncthreads();
        // anticausal: row y uses w[y + 1] (0 for the last row)
        m = make_float2(1.f, 0.f);
#pragma unroll
        for (int i = kDtColRows - 1; i >= 0; --i)
            if (y0 + i < y1) {
                const float w = (i + 1 < kDtColRows && y0 + i + 1 < y1) ? wv[i + 1] : wnx;
                m = amap_compose(make_float2(w, (1.f - w) * iv[i]), m);
            }
        cm[j][col] = m;
        __syncthreads();
#pragma unroll
        for (int r = 1; r < kDtColChunks; r <<= 1) {  // the same in reverse chunk order
            const float2 t = (j + r < kDtColChunks) ? amap_compose(cm[j][col], cm[j + r][col]) : cm[j][col];
            __syncthreads();
            cm[j][col] = t;
            __syncthreads();
        }
        J = (j + 1 < kDtColChunks) ? cm[j + 1][col].y : 0.f;
#pragma unroll
        for (int i = kDtColRows - 1; i >= 0; --i)
            if (y0 + i < y1) {
                const float w = (i + 1 < kDtColRows && y0 + i + 1 < y1) ? wv[i + 1] : wnx;
                J = w * J + (1.f - w) * iv[i];
                cs[(size_t)(y0 + i) * W] = J;
            }
        __syncthreads();
    }
}

}  // namespace fbs
