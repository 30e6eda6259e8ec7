// hier_kernels.cuh — the hierarchical preconditioner and initialisation
// (Eq. hier_precond, hier init PAPER.md:287-293, pyramid PAPER.md:745-766).
//
// P(y) lifts bottom-up and Pᵀ(z) projects top-down through the pyramid (reading #8).  The level
// 0 → 1 lift (≈ M children) runs as a full-occupancy kernel; levels 1..top run in ONE cooperative
// persistent kernel whose large levels are grid-wide phases separated by grid barriers and whose
// coarse levels (≥ 3, a few thousand vertices per frame) are done by one block per frame; the
// level-0 combination of the PCG preconditioner (k_precond_finish2, solve_kernels.cuh) gathers
// the projected level-1 values through the parent map.  Every sum runs over the child lists in
// canonical order, so results are deterministic.
#pragma once
#include "fbs_common.cuh"
#include "solve_kernels.cuh"

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
