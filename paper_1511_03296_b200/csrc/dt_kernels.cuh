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

// d_x = 1 + ratio Σ_c |I_c(x) − I_c(x−1)| (1 at x = 0), d_y likewise; [F][H][W]
__global__ void k_dt_dist(const uint8_t* __restrict__ rgb, int F, int H, int W, float ratio, float* __restrict__ Dx,
                          float* __restrict__ Dy) {
    pdl_entry();
    const int64_t N = (int64_t)F * H * W;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < N; p += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(p % W);
        const int y = (int)((p / W) % H);
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

// out[b][c][r] = in[b][r][c]: 32×32 shared-memory tiles (coalesced both ways)
__global__ void k_transpose(const float* __restrict__ in, int B, int R, int C, float* __restrict__ out) {
    pdl_entry();
    __shared__ float tile[32][33];
    const int64_t tilesC = (C + 31) / 32, tilesR = (R + 31) / 32;
    for (int64_t t = blockIdx.x; t < (int64_t)B * tilesR * tilesC; t += gridDim.x) {
        const int b = (int)(t / (tilesR * tilesC));
        const int tr = (int)((t / tilesC) % tilesR), tc = (int)(t % tilesC);
        const float* src = in + (size_t)b * R * C;
        float* dst = out + (size_t)b * R * C;
        for (int i = threadIdx.y; i < 32; i += blockDim.y) {
            const int r = tr * 32 + i, c = tc * 32 + threadIdx.x;
            if (r < R && c < C) tile[i][threadIdx.x] = src[(size_t)r * C + c];
        }
        __syncthreads();
        for (int i = threadIdx.y; i < 32; i += blockDim.y) {
            const int c = tc * 32 + i, r = tr * 32 + threadIdx.x;
            if (r < R && c < C) dst[(size_t)c * R + r] = tile[threadIdx.x][i];
        }
        __syncthreads();
    }
}

// composition of affine maps J ↦ A J + B: (later ∘ earlier)
__device__ __forceinline__ float2 amap_compose(float2 later, float2 earlier) {
    return make_float2(later.x * earlier.x, later.x * earlier.y + later.y);
}

// One causal + anticausal pass over every line of sig [F][K][Hr][L] (in place), weights
// w = exp(lna · D) with D [F][Hr][L].  Warps per block = blockDim.x / 32; dynamic shared memory:
// 2 · lpad floats per warp, lpad = L + 32 (one pad slot per lane's chunk against bank conflicts).
__global__ void k_dt_rows(float* __restrict__ sig, const float* __restrict__ D, int F, int K, int Hr, int L, float lna) {
    pdl_entry();
    extern __shared__ float dt_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int C = (L + 31) / 32;           // chunk length
    const int lpad = L + 32;               // padded line: element n at n + n / C (lane = n / C ≤ 31)
    float* val = dt_smem + (size_t)warp * 2 * lpad;
    float* wgt = val + lpad;
    const int64_t lines = (int64_t)F * K * Hr;
    for (int64_t r = (int64_t)blockIdx.x * nw + warp; r < lines; r += (int64_t)gridDim.x * nw) {
        const int f = (int)(r / ((int64_t)K * Hr));
        const int y = (int)(r % Hr);
        float* line = sig + (size_t)r * L;
        const float* dl = D + ((size_t)f * Hr + y) * L;
        for (int n = lane; n < L; n += 32) {
            const int pn = n + n / C;
            val[pn] = line[n];
            wgt[pn] = __expf(lna * dl[n]);
        }
        __syncwarp();
        const int n0 = lane * C, n1 = min(n0 + C, L);
        const int base = lane * (C + 1);  // padded index of n0
        // causal: map_n = (w[n], (1 − w[n]) I[n]); element 0 has w = 0
        float2 m = make_float2(1.f, 0.f);
        for (int n = n0, q = base; n < n1; ++n, ++q) {
            const float w = (n == 0) ? 0.f : wgt[q];
            m = amap_compose(make_float2(w, (1.f - w) * val[q]), m);
        }
        float2 incl = m;  // inclusive warp scan (lanes in increasing order)
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const float ax = __shfl_up_sync(0xffffffffu, incl.x, o), ay = __shfl_up_sync(0xffffffffu, incl.y, o);
            if (lane >= o) incl = amap_compose(incl, make_float2(ax, ay));
        }
        float J = __shfl_up_sync(0xffffffffu, incl.y, 1);  // value entering the chunk (maps chain from A = 0)
        for (int n = n0, q = base; n < n1; ++n, ++q) {
            const float w = (n == 0) ? 0.f : wgt[q];
            J = w * J + (1.f - w) * val[q];
            val[q] = J;
        }
        __syncwarp();
        // anticausal: element n uses w[n+1]; the last element keeps its value
        m = make_float2(1.f, 0.f);
        for (int n = n1 - 1; n >= n0; --n) {
            const int q = base + (n - n0);
            const float w = (n == L - 1) ? 0.f : wgt[(n + 1) + (n + 1) / C];
            m = amap_compose(make_float2(w, (1.f - w) * val[q]), m);
        }
        incl = m;  // inclusive scan in decreasing lane order
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const float ax = __shfl_down_sync(0xffffffffu, incl.x, o), ay = __shfl_down_sync(0xffffffffu, incl.y, o);
            if (lane + o < 32) incl = amap_compose(incl, make_float2(ax, ay));
        }
        J = __shfl_down_sync(0xffffffffu, incl.y, 1);
        for (int n = n1 - 1; n >= n0; --n) {
            const int q = base + (n - n0);
            const float w = (n == L - 1) ? 0.f : wgt[(n + 1) + (n + 1) / C];
            J = w * J + (1.f - w) * val[q];
            val[q] = J;
        }
        __syncwarp();
        for (int n = lane; n < L; n += 32) line[n] = val[n + n / C];
        __syncwarp();
    }
}

}  // namespace fbs
