// solve_kernels.cuh — bilateral-space solve on sm_100a.
//
// A is applied in Laplacian-difference form (reading #20):
//   (A y)_v = λ n_v Σ_{u∈N(v)} n_u (y_v − y_u) + Sc_v y_v
// which equals λ(Dm − Dn B̄ Dn) + diag(Sc) at Alg. 1's fixed point n∘B̄n = m.
// It is positive semidefinite by construction in floating point (a weighted graph Laplacian plus
// a non-negative diagonal), keeps constants in the null space of zero-confidence components,
// and its differences (y_v − y_u) are exact for smooth y, so fp32 vectors reach the oracle's
// solution.  Vectors are fp32 planar [K][M]; dots accumulate in fp64 with a fixed-order
// per-frame reduction (block partials + last-block-done), so runs are bitwise reproducible.
// Each (frame, channel) has its own α, β, ρ and stopping rule (reading #13).
#pragma once
#include "fbs_common.cuh"
#include "grid_kernels.cuh"
#include <cooperative_groups.h>

namespace fbs {

struct VecArgs {
    int K, BPF;
    int nf;               // frames of this launch (blocks: nf · BPF); a frame group's VecArgs has
                          // its per-frame pointers shifted to the group's first frame (api.cu)
    int ksplit;           // 1: one channel per block group (F·K·BPF blocks), else F·BPF blocks
    int64_t M;
    float lam;
    const int* frameOff;  // [F+1]
    const int4* nbr;
    const float* n;       // Alg. 1 result
    const float* sc;      // S c
    const float* diagA;   // diag(A) in Laplacian form; 0 ⇔ dead vertex (reading #6)
    float* x;
    float* r;
    float2* dn;           // interleaved (d, n) [K][ldn]: one 8-byte gather per neighbour in the SpMV
    int64_t ldn;          // channel stride of dn: M rounded up to 4 (16-byte aligned bulk copies)
    float* q;
    float* s;
    const float* b;
    const float* mu0;     // level-0 multiplier 1/diag(A) on live vertices (0 on dead ones)
    double* partial;      // [F][BPF][2K]
    unsigned* counters;   // [F][K] last-block counters (block_unit)
    PcgScalars sc_;
    int tol_mode;
    double tol2;
    int max_iters;
};

// Block → (frame f, part j of BPF, channels [k0, k1)) and its last-block counter.  Channel split
// (ksplit): the K right-hand sides of one frame are independent PCGs sharing A, so each gets its
// own BPF blocks — K-fold more parallelism for the multi-channel solves (configs[3]) instead of
// looping the channels inside every block.
struct BlockUnit {
    int f, j, k0, k1;
    int g;  // last-block counter index: f·K + k (split) or f
};
template <int KS>  // 1: split, 0: not split, -1: a.ksplit decides
__device__ __forceinline__ BlockUnit block_unit(const VecArgs& a) {
    BlockUnit u;
    const int g = blockIdx.x / a.BPF;
    u.j = blockIdx.x - g * a.BPF;
    if (KS == 1 || (KS < 0 && a.ksplit)) {
        u.f = g / a.K;
        u.k0 = g - u.f * a.K;
        u.k1 = u.k0 + 1;
    } else {
        u.f = g;
        u.k0 = 0;
        u.k1 = a.K;
    }
    u.g = g;  // non-split: f, unique within a frame group's [f0·K, (f0 + nf)·K)
    return u;
}
__device__ __forceinline__ BlockUnit block_unit(const VecArgs& a) { return block_unit<-1>(a); }

// (A y)_v in Laplacian-difference form (see header): λ n_v Σ_u n_u (y_v − y_u) + Sc_v y_v,
// neighbours in fixed slot order (x−,x+,l−,l+,u−,u+,v−,v+,y−,y+).
__device__ __forceinline__ float apply_A_row(const float* __restrict__ y, const float* __restrict__ n, int v,
                                            int4 nb, float lam, float scv, float yv, float nv) {
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int o = near_off(nb, i);
        if (o) acc += __ldg(n + v + o) * (yv - __ldg(y + v + o));
    }
    if (nb.z) acc += __ldg(n + v + nb.z) * (yv - __ldg(y + v + nb.z));
    if (nb.w) acc += __ldg(n + v + nb.w) * (yv - __ldg(y + v + nb.w));
    return lam * nv * acc + scv * yv;
}
__device__ __forceinline__ float apply_A_row(const float* __restrict__ y, const float* __restrict__ n, int v,
                                            int4 nb, float lam, float scv) {
    return apply_A_row(y, n, v, nb, lam, scv, y[v], n[v]);
}

// Σ_{u∈N(v)} n_u  (so that diag(A) = λ n_v Σ n_u + Sc_v)
__device__ __forceinline__ float nbr_nsum(const float* __restrict__ n, int v, int4 nb) { return nbr_sum(n, v, nb); }

// ---------------------------------------------------------------- splat  S p
// Segment sums in fp32 in a fixed order ("fp32 sums in fixed order"); a
// vertex sums ≤ 64 pixels.  -DFBS_SPLAT_F64 sums in fp64 instead (197 vs 165 µs for the bench batch).
#ifdef FBS_SPLAT_F64
using SplatAcc = double;
#else
using SplatAcc = float;
#endif
// One warp per σxy cell.  The grid build stored each cell's pixels in sorted (code, pixel) order
// (perm), so the pixels of one vertex are consecutive: each vertex sum is a warp segmented scan
// (SplatAcc: fp32, or fp64 with -DFBS_SPLAT_F64) over the two 32-pixel halves, the halves added
// in fixed order — deterministic.  The
// tail lane of each segment writes the vertex sum; the one vertex that may span the halves gets
// half 0's partial (lane 31) carried into half 1's sum.  All of a pixel's loads (vid, c, the
// first channel) go out in one round trip; later channels are prefetched one ahead.
// WEIGHTED: Sc = S c and b_k = S(c∘t_k) (Eq. quad_min); otherwise out_k = S p_k.
template <bool WEIGHTED>
__global__ void __launch_bounds__(256, 8) k_splat(CellGeom g, const int* __restrict__ cellOff,
                                               const unsigned long long* __restrict__ heads,
                                               const uint8_t* __restrict__ perm,
                                               const float* __restrict__ c, const float* __restrict__ p, int K,
                                               int64_t M, float* __restrict__ sc_out, float* __restrict__ out,
                                               int* __restrict__ flags) {
    pdl_entry();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ncells = (int64_t)g.F * g.ncx * g.ncy;
    const size_t HW = (size_t)g.H * g.W;
    for (int cell = blockIdx.x * kCellsPerBlock + warp; cell < (int)ncells;  // cells ≤ pixels < 2^31
         cell += gridDim.x * kCellsPerBlock) {
        int f, cy, cx;
        cell_of(g, cell, f, cy, cx);
        const int x0 = g.colStart[cx], y0 = g.rowStart[cy];
        const int w = g.colStart[cx + 1] - x0, h = g.rowStart[cy + 1] - y0;
        const int npx = min(w * h, kCellMaxPx);
        const unsigned long long H64 = heads[cell];  // run heads of the sorted pixels (k_grid_sort)
        const int vbeg = cellOff[cell];
        const float* pf = p + (size_t)f * K * HW;
        int pix[2], rk[2];
        float cw[2], pv[2];
        bool tail[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int e = lane + 32 * j;
            rk[j] = -1;
            pix[j] = 0;
            cw[j] = 0.f;
            pv[j] = 0.f;
            if (e < npx) {
                const int i = perm[(size_t)cell * kCellMaxPx + e];  // row·8 + column in the cell
                pix[j] = (y0 + (i >> 3)) * g.W + (x0 + (i & 7));
                // the vertex of sorted position e within the cell: its run's rank (= vid − cellOff),
                // from the head mask instead of a gathered vid load
                const unsigned long long upto = (e == 63) ? ~0ull : ((2ull << e) - 1ull);
                rk[j] = __popcll(H64 & upto) - 1;
                cw[j] = WEIGHTED ? c[(size_t)f * HW + pix[j]] : 1.f;
                if (K > 0) pv[j] = pf[pix[j]];
            }
        }
        if (flags) {  // input checks (status bits of fbs_system_stats): c < 0, non-finite c or t
            int bad = 0;
#pragma unroll
            for (int j = 0; j < 2; ++j)
                if (rk[j] >= 0) {
                    if (WEIGHTED && cw[j] < 0.f) bad |= FBS_ST_NEG_CONF;
                    if (!isfinite(cw[j]) || !isfinite(pv[j])) bad |= FBS_ST_NONFINITE;
                }
            bad = __reduce_or_sync(0xffffffffu, bad);
            if (bad && lane == 0) atomicOr(flags, bad);
        }
        // segment bounds inside each half: lane l's segment starts at the last head ≤ l
        int sstart[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int prev = __shfl_up_sync(0xffffffffu, rk[j], 1);
            const bool head = (lane == 0) || (rk[j] != prev);
            const unsigned hm = __ballot_sync(0xffffffffu, head) & ((lane == 31) ? 0xffffffffu : ((2u << lane) - 1u));
            sstart[j] = 31 - __clz(hm);
            const int nxt = __shfl_down_sync(0xffffffffu, rk[j], 1);
            tail[j] = (lane == 31) || (rk[j] != nxt);
        }
        // the vertex spanning the halves: half 0's last segment continues at half 1's lane 0
        const int rk31 = __shfl_sync(0xffffffffu, rk[0], 31);
        const int rk32 = __shfl_sync(0xffffffffu, rk[1], 0);
        const bool span = rk31 >= 0 && rk31 == rk32;
        const int nch = WEIGHTED ? K + 1 : K;
        for (int ch = 0; ch < nch; ++ch) {
            const int k = WEIGHTED ? ch - 1 : ch;  // channel WEIGHTED&&ch==0: Sc; else b_k
            float pn[2] = {0.f, 0.f};
            const bool data = !(WEIGHTED && ch == 0);
            if (data && k + 1 < K) {  // prefetch the next channel
#pragma unroll
                for (int j = 0; j < 2; ++j)
                    if (rk[j] >= 0) pn[j] = pf[(size_t)(k + 1) * HW + pix[j]];
            }
            if (flags && data && k > 0) {  // the later channels' targets
                int bad = 0;
#pragma unroll
                for (int j = 0; j < 2; ++j)
                    if (rk[j] >= 0 && !isfinite(pv[j])) bad = FBS_ST_NONFINITE;
                bad = __reduce_or_sync(0xffffffffu, bad);
                if (bad && lane == 0) atomicOr(flags, bad);
            }
            SplatAcc vs[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                SplatAcc v = 0;
                if (rk[j] >= 0) v = data ? (WEIGHTED ? (SplatAcc)cw[j] * (SplatAcc)pv[j] : (SplatAcc)pv[j]) : (SplatAcc)cw[j];
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {  // segmented inclusive scan (fixed tree)
                    const SplatAcc t = __shfl_up_sync(0xffffffffu, v, d);
                    if (lane - d >= sstart[j]) v += t;
                }
                vs[j] = v;
            }
            const SplatAcc carry = __shfl_sync(0xffffffffu, vs[0], 31);
            float* dst = data ? out + (size_t)k * M + vbeg : sc_out + vbeg;
            if (tail[0] && rk[0] >= 0 && !(lane == 31 && span)) dst[rk[0]] = (float)(vs[0]);
            if (tail[1] && rk[1] >= 0) dst[rk[1]] = (float)((span && sstart[1] == 0) ? carry + vs[1] : vs[1]);
            if (data) {
                pv[0] = pn[0];
                pv[1] = pn[1];
            }
        }
    }
}

// ---------------------------------------------------------------- per-frame reductions
// Alg. 2 lines 11-13 + stopping rule (reading #11) for one (frame, channel) given its reduced
// ρ = rᵀs and ‖r‖²; executed by one thread.  first: the reduction right after initialisation
// (lines 2-4).
__device__ __forceinline__ void finish_rho_one(const VecArgs& a, int fk, bool first, double R, double RR) {
    const bool conv = a.tol_mode && RR <= a.tol2 * a.sc_.bb[fk];
    a.sc_.rr[fk] = RR;
    if (first) {
        a.sc_.rho[fk] = R;
        a.sc_.beta[fk] = 0.0;
        a.sc_.iters[fk] = 0;
        const bool act = !conv && R != 0.0 && a.max_iters > 0;
        a.sc_.active[fk] = act;
        if (!act) atomicSub(a.sc_.n_active, 1);
    } else {
        a.sc_.beta[fk] = R / a.sc_.rho[fk];
        a.sc_.rho[fk] = R;
        const int it = a.sc_.iters[fk] + 1;
        a.sc_.iters[fk] = it;
        if (conv || R == 0.0 || it >= a.max_iters) {
            if (!conv && a.tol_mode && R != 0.0) atomicOr(a.sc_.status + fk, FBS_ST_NOTCONVERGED);
            a.sc_.active[fk] = 0;
            atomicSub(a.sc_.n_active, 1);
        }
    }
}

// finish of the ρ-reduction executed by the last block of frame f (partials [F][BPF][2K]).
__device__ void finish_rho(const VecArgs& a, int f, int k0, int k1, bool first, double* shd) {
    for (int k = k0; k < k1; ++k) {
        const int fk = f * a.K + k;
        if (!first && !a.sc_.active[fk]) continue;
        double R = 0.0, RR = 0.0;
        for (int j = threadIdx.x; j < a.BPF; j += blockDim.x) {
            const double* pp = a.partial + ((size_t)f * a.BPF + j) * 2 * a.K + 2 * k;
            R += __ldcg(pp);
            RR += __ldcg(pp + 1);
        }
        block_sum2(R, RR, shd);
        if (threadIdx.x == 0) finish_rho_one(a, fk, first, R, RR);
    }
}

// (ONE: v1 is 0 and needs no reduction)
template <bool ONE = false>
__device__ __forceinline__ void write_partials(const VecArgs& a, int f, int j, int k, double v0, double v1,
                                               double* shd) {
    if (ONE) v0 = block_sum(v0, shd);
    else block_sum2(v0, v1, shd);
    if (threadIdx.x == 0) {
        double* pp = a.partial + ((size_t)f * a.BPF + j) * 2 * a.K + 2 * k;
        pp[0] = v0;
        pp[1] = v1;
    }
}

// ---------------------------------------------------------------- assemble (Eq. quad_min)
// diag(A) = λ n_v Σ_u n_u + Sc_v (PAPER.md:230 at Alg. 1's fixed point; isolated vertex: Sc_v,
// reading #6), μ0 = 1/diag(A) on live vertices (Jacobi), ‖b‖² per (frame, k),
// flat init y_flat = b/Sc (reading #9) or zero init, and the interleaved (d, n)
// vector with d = 0.  Per-frame blocks.
__global__ void __launch_bounds__(256) k_assemble(VecArgs a, float* __restrict__ diagA, float* __restrict__ mu0,
                                                  int init_mode, PcgScalars scal) {
    pdl_entry();
    __shared__ double shd[32];
    __shared__ int sflag;
    const BlockUnit bu = block_unit(a);
    const int f = bu.f, j = bu.j;
    const int v0 = a.frameOff[f], v1 = a.frameOff[f + 1];
    for (int v = v0 + j * blockDim.x + threadIdx.x; bu.k0 == 0 && v < v1; v += a.BPF * blockDim.x) {
        const float dA = a.lam * a.n[v] * nbr_nsum(a.n, v, a.nbr[v]) + a.sc[v];
        const bool live = dA > 0.f;
        diagA[v] = dA;
        mu0[v] = live ? 1.f / dA : 0.f;
    }
    for (int k = bu.k0; k < bu.k1; ++k) {
        double bb = 0.0;
        const size_t off = (size_t)k * a.M;
        for (int v = v0 + j * blockDim.x + threadIdx.x; v < v1; v += a.BPF * blockDim.x) {
            const float b = a.b[off + v];
            bb += (double)b * (double)b;
            a.dn[(size_t)k * a.ldn + v] = make_float2(0.f, a.n[v]);  // (d, n) with d = 0
            if (init_mode == FBS_INIT_FLAT) {
                const float S = a.sc[v];
                a.x[off + v] = (S > 0.f) ? b / S : 0.f;
            } else if (init_mode == FBS_INIT_ZERO) {
                a.x[off + v] = 0.f;
            }
        }
        write_partials<true>(a, f, j, k, bb, 0.0, shd);
    }
    if (last_block_t0(a.counters + bu.g, a.BPF, &sflag)) {
        for (int k = bu.k0; k < bu.k1; ++k) {
            double R = 0.0;
            for (int jj = threadIdx.x; jj < a.BPF; jj += blockDim.x)
                R += __ldcg(a.partial + ((size_t)f * a.BPF + jj) * 2 * a.K + 2 * k);
            R = block_sum(R, shd);
            if (threadIdx.x == 0) scal.bb[f * a.K + k] = R;
        }
    }
}

// ---------------------------------------------------------------- hierarchical init input [b_0..b_{K−1}, Sc]
__global__ void k_fill_init_w0(const float* __restrict__ b, const float* __restrict__ sc, int64_t M, int K,
                               float* __restrict__ w0) {
    pdl_entry();
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < M; v += (int64_t)gridDim.x * blockDim.x) {
        for (int k = 0; k < K; ++k) w0[(size_t)k * M + v] = b[(size_t)k * M + v];
        w0[(size_t)K * M + v] = sc[v];
    }
}

// ---------------------------------------------------------------- PCG (Alg. 2)
// scalars of n (frame, channel) pairs (a frame group's arrays are pointer-shifted); set_count:
// also the global active count of the TOL-mode host poll
__global__ void k_init_scalars(PcgScalars s, int n, int set_count) {
    pdl_entry();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        s.rho[i] = 0.0;
        s.alpha[i] = 0.0;
        s.xalpha[i] = 0.0;
        s.beta[i] = 0.0;
        s.rr[i] = 0.0;
        s.active[i] = 1;
        s.iters[i] = 0;
        s.status[i] = 0;
    }
    if (i == 0 && set_count) *s.n_active = n;
}

// Alg. 2 lines 2-4 (Jacobi):  r = b − A x;  s = M⁻¹ r;  ρ = rᵀs   (X_ZERO: x = 0 ⇒ r = b, backward).
// The hierarchical preconditioner has its own fused kernels (tile_kernels.cuh).
template <bool X_ZERO>
__global__ void __launch_bounds__(256) k_residual0(VecArgs a) {
    pdl_entry();
    __shared__ double shd[32];
    __shared__ int sflag;
    const BlockUnit bu = block_unit(a);
    const int f = bu.f, j = bu.j;
    const int v0 = a.frameOff[f], v1 = a.frameOff[f + 1];
    for (int k = bu.k0; k < bu.k1; ++k) {
        const size_t off = (size_t)k * a.M;
        double rho = 0.0, rr = 0.0;
        for (int v = v0 + j * blockDim.x + threadIdx.x; v < v1; v += a.BPF * blockDim.x) {
            float r = a.b[off + v];
            if (!X_ZERO) r -= apply_A_row(a.x + off, a.n, v, a.nbr[v], a.lam, a.sc[v]);
            a.r[off + v] = r;
            const float s = a.mu0[v] * r;
            a.s[off + v] = s;
            rho += (double)r * (double)s;
            rr += (double)r * (double)r;
        }
        write_partials(a, f, j, k, rho, rr, shd);
    }
    if (last_block_t0(a.counters + bu.g, a.BPF, &sflag)) finish_rho(a, f, bu.k0, bu.k1, true, shd);
}

// Alg. 2 lines 8-12 (Jacobi):  x += αd;  r −= αq;  s = M⁻¹r = r/diag(A);  ρ_new = rᵀs.
__global__ void __launch_bounds__(256, 8) k_update(VecArgs a) {
    pdl_entry();
    __shared__ double shd[32];
    __shared__ int sflag;
    const BlockUnit bu = block_unit(a);
    const int f = bu.f, j = bu.j;
    const int v0 = a.frameOff[f], v1 = a.frameOff[f + 1];
    for (int k = bu.k0; k < bu.k1; ++k) {
        const int fk = f * a.K + k;
        double rho = 0.0, rr = 0.0;
        if (a.sc_.active[fk]) {
            const float al = (float)a.sc_.alpha[fk];
            const size_t off = (size_t)k * a.M;
            const int stride = a.BPF * blockDim.x;
            for (int v0u = v0 + j * blockDim.x + threadIdx.x; v0u < v1; v0u += 4 * stride) {
                // loads of 4 vertices first (the VecArgs pointers may alias for the compiler)
                float xv[4], dv[4], rv[4], qv[4], mv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int v = v0u + u * stride;
                    if (v < v1) {
                        xv[u] = a.x[off + v];
                        dv[u] = a.dn[(size_t)k * a.ldn + v].x;
                        rv[u] = a.r[off + v];
                        qv[u] = a.q[off + v];
                        mv[u] = a.mu0[v];
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int v = v0u + u * stride;
                    if (v >= v1) continue;
                    a.x[off + v] = xv[u] + al * dv[u];
                    const float r = rv[u] - al * qv[u];
                    a.r[off + v] = r;
                    const float s = mv[u] * r;
                    a.s[off + v] = s;
                    rho += (double)r * (double)s;
                    rr += (double)r * (double)r;
                }
            }
        }
        write_partials(a, f, j, k, rho, rr, shd);
    }
    if (last_block_t0(a.counters + bu.g, a.BPF, &sflag)) finish_rho(a, f, bu.k0, bu.k1, false, shd);
}

// ---------------------------------------------------------------- small systems: Alg. 2 in one CTA
// A frame of ≤ kSmallPx pixels (configs[0]-sized) has a few thousand vertices: each multi-kernel
// PCG iteration is three ~4 µs launches plus, in TOL mode, host polls.  Here one CTA runs the
// whole Jacobi PCG of one (frame, channel) — Alg. 2 lines 2-4, then per iteration lines 14, 6-7,
// 8-12 — with block barriers in place of kernel boundaries (the vectors stay in L1/L2) and the
// stopping rule on the device.  Per-vertex arithmetic, the fp32 casts of α and β and the scalar
// recurrences / stopping rule (finish_rho_one) are those of k_residual0 / k_direction2 / k_spmv2 /
// k_update; only the fp64 dot products' summation order differs (one block's tree).
constexpr int kSmallThreads = 512;  // block_sum2 holds ≤ 16 warps
constexpr int kSmallPx = 8192;      // default per-frame pixel bound of the one-CTA path (api.cu run_pcg)
__global__ void __launch_bounds__(kSmallThreads) k_pcg_small(VecArgs a, int x_zero) {
    pdl_entry();
    __shared__ double shd[32];
    __shared__ double s_beta;
    __shared__ float s_alpha;
    __shared__ int s_active;
    const int f = blockIdx.x / a.K, k = blockIdx.x - f * a.K;
    const int fk = f * a.K + k;
    const int v0 = a.frameOff[f], v1 = a.frameOff[f + 1];
    const size_t off = (size_t)k * a.M;
    float* __restrict__ x = a.x + off;
    float* __restrict__ r = a.r + off;
    float* __restrict__ s = a.s + off;
    float* __restrict__ q = a.q + off;
    float2* __restrict__ dn = a.dn + (size_t)k * a.ldn;
    // Alg. 2 lines 2-4: r = b − A x, s = M⁻¹r, ρ = rᵀs
    double R = 0.0, RR = 0.0;
    for (int v = v0 + threadIdx.x; v < v1; v += blockDim.x) {
        float rv = a.b[off + v];
        if (!x_zero) rv -= apply_A_row(x, a.n, v, a.nbr[v], a.lam, a.sc[v]);
        r[v] = rv;
        const float sv = a.mu0[v] * rv;
        s[v] = sv;
        R += (double)rv * (double)sv;
        RR += (double)rv * (double)rv;
    }
    block_sum2(R, RR, shd);
    if (threadIdx.x == 0) {
        finish_rho_one(a, fk, true, R, RR);
        s_active = a.sc_.active[fk];
        s_beta = 0.0;
    }
    __syncthreads();
    for (int it = 0; s_active; ++it) {
        // line 14 (line 3 at it = 0): d = s + βd
        const float be = (float)s_beta;
        for (int v = v0 + threadIdx.x; v < v1; v += blockDim.x) {
            const float2 dv = dn[v];
            dn[v] = make_float2(it == 0 ? s[v] : s[v] + be * dv.x, dv.y);
        }
        __syncthreads();
        // lines 6-7: q = A d (Laplacian-difference form), α = ρ / dᵀq
        double dq = 0.0;
        for (int v = v0 + threadIdx.x; v < v1; v += blockDim.x) {
            const int4 nb = a.nbr[v];
            const float2 me = dn[v];
            float acc = 0.f;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int o = near_off(nb, e);
                if (o) {
                    const float2 u = dn[v + o];
                    acc += u.y * (me.x - u.x);
                }
            }
            if (nb.z) {
                const float2 u = dn[v + nb.z];
                acc += u.y * (me.x - u.x);
            }
            if (nb.w) {
                const float2 u = dn[v + nb.w];
                acc += u.y * (me.x - u.x);
            }
            const float qv = a.lam * me.y * acc + a.sc[v] * me.x;
            q[v] = qv;
            dq += (double)me.x * (double)qv;
        }
        dq = block_sum(dq, shd);
        if (threadIdx.x == 0) {
            if (dq <= 0.0) {
                a.sc_.active[fk] = 0;
                a.sc_.alpha[fk] = 0.0;
                a.sc_.xalpha[fk] = 0.0;
                atomicOr(a.sc_.status + fk, FBS_ST_BREAKDOWN);
                atomicSub(a.sc_.n_active, 1);
                s_active = 0;
            } else {
                const double al = a.sc_.rho[fk] / dq;
                a.sc_.alpha[fk] = al;
                a.sc_.xalpha[fk] = al;
                s_alpha = (float)al;
            }
        }
        __syncthreads();
        if (!s_active) break;
        // lines 8-12: x += αd, r −= αq, s = M⁻¹r, ρ_new = rᵀs (and ‖r‖² for the stopping rule)
        const float al = s_alpha;
        R = 0.0;
        RR = 0.0;
        for (int v = v0 + threadIdx.x; v < v1; v += blockDim.x) {
            x[v] = x[v] + al * dn[v].x;
            const float rv = r[v] - al * q[v];
            r[v] = rv;
            const float sv = a.mu0[v] * rv;
            s[v] = sv;
            R += (double)rv * (double)sv;
            RR += (double)rv * (double)rv;
        }
        block_sum2(R, RR, shd);
        if (threadIdx.x == 0) {
            finish_rho_one(a, fk, false, R, RR);
            s_active = a.sc_.active[fk];
            s_beta = a.sc_.beta[fk];
        }
        __syncthreads();
    }
}

// Medium frames: the same one-launch Jacobi PCG with a cluster of kPcgCluster CTAs per (frame,
// channel).  Vertex v of the frame belongs to CTA rank (v − v0) / blockDim mod kPcgCluster; a
// phase's dot product is each CTA's block tree, its partial left in shared memory, then summed by
// every CTA over the cluster's ranks in rank order through distributed shared memory — the same
// value in every CTA, so each CTA takes the same α, β and stopping decision (rank 0 alone writes
// the global scalars through finish_rho_one).  Three cluster barriers per iteration (after the
// direction: the SpMV gathers other CTAs' d; after each reduction); the (d, n) vector, shared
// across CTAs, goes through L2 (ld/st.cg), the per-vertex vectors stay with their owner thread.
#ifndef FBS_CLUSTER_MINB
#define FBS_CLUSTER_MINB 2  // resident CTAs per SM the register budget allows (A/B: -DFBS_CLUSTER_MINB=3)
#endif
constexpr int kPcgCluster = 8;
constexpr int kClusterPx = 262144;  // default per-frame pixel bound of the cluster path (api.cu run_pcg)
constexpr int kClusterPxAnyK = 98304;  // ... for any (frame, channel) count; above it ≥ 16 of them
__global__ void __cluster_dims__(kPcgCluster, 1, 1) __launch_bounds__(kSmallThreads, FBS_CLUSTER_MINB)
    k_pcg_cluster(VecArgs a, int x_zero) {
    namespace cg = cooperative_groups;
    pdl_entry();
    cg::cluster_group cl = cg::this_cluster();
    __shared__ double shd[32];
    __shared__ double part[2][2];  // [slot][value]: slot 0 the SpMV's dᵀq, slot 1 (ρ, ‖r‖²)
    const int rank = (int)cl.block_rank();
    const int u = blockIdx.x / kPcgCluster;
    const int f = u / a.K, k = u - f * a.K;
    const int fk = f * a.K + k;
    const int v0 = a.frameOff[f], v1 = a.frameOff[f + 1];
    const int vbeg = v0 + rank * blockDim.x + threadIdx.x, stride = kPcgCluster * blockDim.x;
    const size_t off = (size_t)k * a.M;
    float* __restrict__ x = a.x + off;
    float* __restrict__ r = a.r + off;
    float* __restrict__ s = a.s + off;
    float* __restrict__ q = a.q + off;
    float2* dn = a.dn + (size_t)k * a.ldn;
    // cluster-wide sums of slot `sl` (after the barrier that published every CTA's partial)
    auto cluster_sum = [&](int sl, double& s0, double& s1) {
        s0 = 0.0;
        s1 = 0.0;
        for (int q2 = 0; q2 < kPcgCluster; ++q2) {
            const double* p = cl.map_shared_rank(&part[sl][0], q2);
            s0 += p[0];
            s1 += p[1];
        }
    };
    const double bb = a.sc_.bb[fk];
    // Alg. 2 lines 2-4
    double R = 0.0, RR = 0.0;
    for (int v = vbeg; v < v1; v += stride) {
        float rv = a.b[off + v];
        if (!x_zero) rv -= apply_A_row(x, a.n, v, a.nbr[v], a.lam, a.sc[v]);
        r[v] = rv;
        const float sv = a.mu0[v] * rv;
        s[v] = sv;
        R += (double)rv * (double)sv;
        RR += (double)rv * (double)rv;
    }
    block_sum2(R, RR, shd);
    if (threadIdx.x == 0) {
        part[1][0] = R;
        part[1][1] = RR;
    }
    cl.sync();
    cluster_sum(1, R, RR);
    if (rank == 0 && threadIdx.x == 0) finish_rho_one(a, fk, true, R, RR);
    double rho = R;
    bool active = !(a.tol_mode && RR <= a.tol2 * bb) && R != 0.0 && a.max_iters > 0;
    double beta = 0.0;
    for (int it = 0; active; ++it) {
        const float be = (float)beta;
        for (int v = vbeg; v < v1; v += stride) {
            const float2 dv = __ldcg(dn + v);
            __stcg(dn + v, make_float2(it == 0 ? s[v] : s[v] + be * dv.x, dv.y));
        }
        cl.sync();
        double dq = 0.0;
        for (int v = vbeg; v < v1; v += stride) {
            const int4 nb = a.nbr[v];
            const float2 me = __ldcg(dn + v);
            float acc = 0.f;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int o = near_off(nb, e);
                if (o) {
                    const float2 w = __ldcg(dn + v + o);
                    acc += w.y * (me.x - w.x);
                }
            }
            if (nb.z) {
                const float2 w = __ldcg(dn + v + nb.z);
                acc += w.y * (me.x - w.x);
            }
            if (nb.w) {
                const float2 w = __ldcg(dn + v + nb.w);
                acc += w.y * (me.x - w.x);
            }
            const float qv = a.lam * me.y * acc + a.sc[v] * me.x;
            q[v] = qv;
            dq += (double)me.x * (double)qv;
        }
        dq = block_sum(dq, shd);
        if (threadIdx.x == 0) {
            part[0][0] = dq;
            part[0][1] = 0.0;
        }
        cl.sync();
        double DQ, unused;
        cluster_sum(0, DQ, unused);
        if (DQ <= 0.0) {
            if (rank == 0 && threadIdx.x == 0) {
                a.sc_.active[fk] = 0;
                a.sc_.alpha[fk] = 0.0;
                a.sc_.xalpha[fk] = 0.0;
                atomicOr(a.sc_.status + fk, FBS_ST_BREAKDOWN);
                atomicSub(a.sc_.n_active, 1);
            }
            break;
        }
        const double alpha = rho / DQ;
        if (rank == 0 && threadIdx.x == 0) {
            a.sc_.alpha[fk] = alpha;
            a.sc_.xalpha[fk] = alpha;
        }
        const float al = (float)alpha;
        R = 0.0;
        RR = 0.0;
        for (int v = vbeg; v < v1; v += stride) {
            x[v] = x[v] + al * __ldcg(dn + v).x;
            const float rv = r[v] - al * q[v];
            r[v] = rv;
            const float sv = a.mu0[v] * rv;
            s[v] = sv;
            R += (double)rv * (double)sv;
            RR += (double)rv * (double)rv;
        }
        block_sum2(R, RR, shd);
        if (threadIdx.x == 0) {
            part[1][0] = R;
            part[1][1] = RR;
        }
        cl.sync();
        cluster_sum(1, R, RR);
        if (rank == 0 && threadIdx.x == 0) finish_rho_one(a, fk, false, R, RR);
        // finish_rho_one's recurrence and stopping rule, taken identically by every CTA
        beta = R / rho;
        rho = R;
        const bool conv = a.tol_mode && RR <= a.tol2 * bb;
        if (conv || R == 0.0 || it + 1 >= a.max_iters) active = false;
    }
    cl.sync();  // no CTA exits while another may still read its partials
}

// ---------------------------------------------------------------- streaming PCG kernels
// dn[k][v] = (d, n_v) (initialised by k_assemble): the direction interleaved with n, so the
// SpMV's neighbour terms n_u (d_v − d_u) need ONE 8-byte gather per neighbour.

// Alg. 2 line 14:  d = s + βd  (first: d = s, line 3).
__global__ void __launch_bounds__(256, 8) k_direction2(VecArgs a, int first) {
    pdl_entry();
    const BlockUnit bu = block_unit(a);
    const int f = bu.f, j = bu.j;
    const int v0 = a.frameOff[f], v1 = a.frameOff[f + 1];
    const int stride = a.BPF * blockDim.x;
    for (int k = bu.k0; k < bu.k1; ++k) {
        const int fk = f * a.K + k;
        if (!first && !a.sc_.active[fk]) continue;
        const float be = first ? 0.f : (float)a.sc_.beta[fk];
        const size_t off = (size_t)k * a.M;
        for (int v0u = v0 + j * blockDim.x + threadIdx.x; v0u < v1; v0u += 4 * stride) {
            float sv[4];
            float2 dv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int v = v0u + u * stride;
                if (v < v1) {
                    sv[u] = a.s[off + v];
                    dv[u] = a.dn[(size_t)k * a.ldn + v];
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int v = v0u + u * stride;
                if (v < v1) a.dn[(size_t)k * a.ldn + v] = make_float2(first ? sv[u] : sv[u] + be * dv[u].x, dv[u].y);
            }
        }
    }
}

// Alg. 2 lines 6-7:  q = A d (Laplacian-difference form), α = ρ / dᵀq (breakdown: dᵀq ≤ 0).
// Latency-bound gathers: 8 resident blocks per SM (≤ 32 registers) matter (40 registers: 6 blocks,
// 45 → 68 µs on the bench workload with one frame group), and ptxas's allocation for this loop is
// fragile, so the unsplit kernel keeps its own body and the channel-split one (K > 1) has its own.
__global__ void __launch_bounds__(256) k_spmv2(VecArgs a) {
    pdl_entry();
    __shared__ double shd[32];
    __shared__ int sflag;
    const int f = blockIdx.x / a.BPF, j = blockIdx.x % a.BPF;
    const int v0 = a.frameOff[f], v1 = a.frameOff[f + 1];
    for (int k = 0; k < a.K; ++k) {
        const int fk = f * a.K + k;
        double dq = 0.0;
        if (a.sc_.active[fk]) {
            const size_t off = (size_t)k * a.M;
            const float2* dn = a.dn + (size_t)k * a.ldn;
            for (int v = v0 + j * blockDim.x + threadIdx.x; v < v1; v += a.BPF * blockDim.x) {
                const int4 nb = __ldcs(a.nbr + v);  // streamed once per iteration: evict-first
                const float2 me = dn[v];
                const float scv = __ldcs(a.sc + v);
                float acc = 0.f;
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int o = near_off(nb, e);
                    if (o) {
                        const float2 u = __ldg(dn + v + o);
                        acc += u.y * (me.x - u.x);
                    }
                }
                if (nb.z) {
                    const float2 u = __ldg(dn + v + nb.z);
                    acc += u.y * (me.x - u.x);
                }
                if (nb.w) {
                    const float2 u = __ldg(dn + v + nb.w);
                    acc += u.y * (me.x - u.x);
                }
                const float q = a.lam * me.y * acc + scv * me.x;
                a.q[off + v] = q;
                dq += (double)me.x * (double)q;
            }
        }
        write_partials<true>(a, f, j, k, dq, 0.0, shd);
    }
    if (last_block_t0(a.counters + f, a.BPF, &sflag)) {
        for (int k = 0; k < a.K; ++k) {
            const int fk = f * a.K + k;
            if (!a.sc_.active[fk]) {
                if (threadIdx.x == 0) a.sc_.xalpha[fk] = 0.0;
                continue;
            }
            double DQ = 0.0;
            for (int jj = threadIdx.x; jj < a.BPF; jj += blockDim.x)
                DQ += __ldcg(a.partial + ((size_t)f * a.BPF + jj) * 2 * a.K + 2 * k);
            DQ = block_sum(DQ, shd);
            if (threadIdx.x == 0) {
                if (DQ <= 0.0) {
                    a.sc_.active[fk] = 0;
                    a.sc_.alpha[fk] = 0.0;
                    a.sc_.xalpha[fk] = 0.0;
                    atomicOr(a.sc_.status + fk, FBS_ST_BREAKDOWN);
                    atomicSub(a.sc_.n_active, 1);
                } else {
                    a.sc_.alpha[fk] = a.sc_.rho[fk] / DQ;
                    a.sc_.xalpha[fk] = a.sc_.alpha[fk];
                }
            }
        }
    }
}

// q_k = A d_k for all K channels of a frame with ONE read of the neighbour structure per vertex
// (north_star: "K-channel right-hand sides are solved jointly, sharing one neighbour-index
// read"): a warp per vertex, a lane per channel (k = lane, lane + 32).  The warp's 16-byte nbr
// and Sc loads are one broadcast transaction; each lane gathers its own channel's (d, n).  dᵀq_k
// partials: per lane in registers, then a fixed-order sum over the block's warps (deterministic);
// the last block of the frame finishes every channel's α as k_spmv2 does.
__global__ void __launch_bounds__(256) k_spmv_kjoint(VecArgs a) {
    pdl_entry();
    __shared__ double sdq[kThreads / 32][kMaxK];
    __shared__ double shd[32];
    __shared__ int sflag;
    const int f = blockIdx.x / a.BPF, j = blockIdx.x % a.BPF;
    const int v0 = a.frameOff[f], v1 = a.frameOff[f + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int WPB = kThreads / 32;
    double dq[2] = {0.0, 0.0};
    bool act[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int k = lane + 32 * h;
        act[h] = k < a.K && a.sc_.active[f * a.K + k];
    }
    for (int v = v0 + j * WPB + warp; v < v1; v += a.BPF * WPB) {
        const int4 nb = __ldcs(a.nbr + v);  // the same address in every lane: one transaction
        const float scv = __ldcs(a.sc + v);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (!act[h]) continue;
            const int k = lane + 32 * h;
            const float2* dn = a.dn + (size_t)k * a.ldn;
            const float2 me = dn[v];
            float acc = 0.f;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int o = near_off(nb, e);
                if (o) {
                    const float2 u = __ldg(dn + v + o);
                    acc += u.y * (me.x - u.x);
                }
            }
            if (nb.z) {
                const float2 u = __ldg(dn + v + nb.z);
                acc += u.y * (me.x - u.x);
            }
            if (nb.w) {
                const float2 u = __ldg(dn + v + nb.w);
                acc += u.y * (me.x - u.x);
            }
            const float q = a.lam * me.y * acc + scv * me.x;
            a.q[(size_t)k * a.M + v] = q;
            dq[h] += (double)me.x * (double)q;
        }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h)
        if (lane + 32 * h < a.K) sdq[warp][lane + 32 * h] = dq[h];
    __syncthreads();
    for (int k = threadIdx.x; k < a.K; k += blockDim.x) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < WPB; ++w) t += sdq[w][k];
        a.partial[((size_t)f * a.BPF + j) * 2 * a.K + 2 * k] = t;
    }
    if (last_block_of_frame(a.counters + f, a.BPF, &sflag)) {
        for (int k = 0; k < a.K; ++k) {
            const int fk = f * a.K + k;
            if (!a.sc_.active[fk]) {
                if (threadIdx.x == 0) a.sc_.xalpha[fk] = 0.0;
                continue;
            }
            double DQ = 0.0;
            for (int jj = threadIdx.x; jj < a.BPF; jj += blockDim.x)
                DQ += __ldcg(a.partial + ((size_t)f * a.BPF + jj) * 2 * a.K + 2 * k);
            DQ = block_sum(DQ, shd);
            if (threadIdx.x == 0) {
                if (DQ <= 0.0) {
                    a.sc_.active[fk] = 0;
                    a.sc_.alpha[fk] = 0.0;
                    a.sc_.xalpha[fk] = 0.0;
                    atomicOr(a.sc_.status + fk, FBS_ST_BREAKDOWN);
                    atomicSub(a.sc_.n_active, 1);
                } else {
                    a.sc_.alpha[fk] = a.sc_.rho[fk] / DQ;
                    a.sc_.xalpha[fk] = a.sc_.alpha[fk];
                }
            }
        }
    }
}

__global__ void __launch_bounds__(256) k_spmv2_split(VecArgs a) {
    pdl_entry();
    __shared__ double shd[32];
    __shared__ int sflag;
    const int g = blockIdx.x / a.BPF, j = blockIdx.x % a.BPF;
    const int f = g / a.K;  // block_unit, inline
    const int kb = g - f * a.K, ke = kb + 1;
    const int v0 = a.frameOff[f], v1 = a.frameOff[f + 1];
    for (int k = kb; k < ke; ++k) {
        const int fk = f * a.K + k;
        double dq = 0.0;
        if (a.sc_.active[fk]) {
            const size_t off = (size_t)k * a.M;
            const float2* dn = a.dn + (size_t)k * a.ldn;
            for (int v = v0 + j * blockDim.x + threadIdx.x; v < v1; v += a.BPF * blockDim.x) {
                const int4 nb = __ldcs(a.nbr + v);  // streamed once per iteration: evict-first
                const float2 me = dn[v];
                const float scv = __ldcs(a.sc + v);
                float acc = 0.f;
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int o = near_off(nb, e);
                    if (o) {
                        const float2 u = __ldg(dn + v + o);
                        acc += u.y * (me.x - u.x);
                    }
                }
                if (nb.z) {
                    const float2 u = __ldg(dn + v + nb.z);
                    acc += u.y * (me.x - u.x);
                }
                if (nb.w) {
                    const float2 u = __ldg(dn + v + nb.w);
                    acc += u.y * (me.x - u.x);
                }
                const float q = a.lam * me.y * acc + scv * me.x;
                a.q[off + v] = q;
                dq += (double)me.x * (double)q;
            }
        }
        write_partials<true>(a, f, j, k, dq, 0.0, shd);
    }
    if (last_block_t0(a.counters + g, a.BPF, &sflag)) {
        for (int k = kb; k < ke; ++k) {
            const int fk = f * a.K + k;
            if (!a.sc_.active[fk]) {
                if (threadIdx.x == 0) a.sc_.xalpha[fk] = 0.0;
                continue;
            }
            double DQ = 0.0;
            for (int jj = threadIdx.x; jj < a.BPF; jj += blockDim.x)
                DQ += __ldcg(a.partial + ((size_t)f * a.BPF + jj) * 2 * a.K + 2 * k);
            DQ = block_sum(DQ, shd);
            if (threadIdx.x == 0) {
                if (DQ <= 0.0) {
                    a.sc_.active[fk] = 0;
                    a.sc_.alpha[fk] = 0.0;
                    a.sc_.xalpha[fk] = 0.0;
                    atomicOr(a.sc_.status + fk, FBS_ST_BREAKDOWN);
                    atomicSub(a.sc_.n_active, 1);
                } else {
                    a.sc_.alpha[fk] = a.sc_.rho[fk] / DQ;
                    a.sc_.xalpha[fk] = a.sc_.alpha[fk];
                }
            }
        }
    }
}

// Condition of the TOL loop: another iteration while any (frame, channel) is active (each
// retires itself at convergence, breakdown or max_iters); `it` bounds it defensively.
__global__ void k_tol_cond(cudaGraphConditionalHandle h, const int* __restrict__ n_active, int* __restrict__ it,
                           int max_body) {
    pdl_entry();  // launched with PDL like every kernel: wait for the iteration's last atomicSub
    if (threadIdx.x == 0) {
        const int i = ++*it;
        cudaGraphSetConditional(h, (*n_active > 0 && i < max_body) ? 1u : 0u);
    }
}

// The host-polled TOL loop's probe (api.cu tol_poll): the active count and, for a single (frame,
// channel), ‖b‖² and the last ‖r‖², into mapped pinned memory laid out as {int, pad, double, double}.
__global__ void k_tol_probe(const int* __restrict__ n_active, const double* __restrict__ bb,
                            const double* __restrict__ rr, int* __restrict__ out) {
    pdl_entry();
    if (threadIdx.x == 0) {
        out[0] = *n_active;
        double* d = reinterpret_cast<double*>(out + 2);
        d[0] = bb ? *bb : 0.0;
        d[1] = rr ? *rr : 0.0;
    }
}

// ---------------------------------------------------------------- slice / export / backward
// x̂ = Sᵀŷ.  ys planar [K][M] (planar = 1) or canonical [M][K].
__global__ void k_slice(const int* __restrict__ vid, const float* __restrict__ ys, int64_t M, int K, int F,
                        int64_t HW, int planar, float* __restrict__ out) {
    pdl_entry();
    const int64_t N = (int64_t)F * HW;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < N; p += (int64_t)gridDim.x * blockDim.x) {
        const int v = vid[p];
        const int f = (int)(p / HW);
        const int64_t pp = p - (int64_t)f * HW;
        for (int k = 0; k < K; ++k) {
            const float y = planar ? ys[(size_t)k * M + v] : ys[(size_t)v * K + k];
            out[((size_t)f * K + k) * HW + pp] = y;
        }
    }
}

// k_slice for HW % 4 == 0 and a 16-byte-aligned output: 4 pixels per thread (one 16-byte vid
// load, 4 independent gathers, one 16-byte store per channel), the frame from blockIdx.y (no
// 64-bit division per pixel).
__global__ void k_slice4(const int* __restrict__ vid, const float* __restrict__ ys, int64_t M, int K, int64_t HW,
                         int planar, float* __restrict__ out) {
    pdl_entry();
    const int f = blockIdx.y;
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i >= HW) return;
    const int4 v = __ldcs(reinterpret_cast<const int4*>(vid + (size_t)f * HW + i));
    for (int k = 0; k < K; ++k) {
        float4 y;
        if (planar) {
            const float* yk = ys + (size_t)k * M;
            y = make_float4(yk[v.x], yk[v.y], yk[v.z], yk[v.w]);
        } else {
            y = make_float4(ys[(size_t)v.x * K + k], ys[(size_t)v.y * K + k], ys[(size_t)v.z * K + k],
                            ys[(size_t)v.w * K + k]);
        }
        __stcs(reinterpret_cast<float4*>(out + ((size_t)f * K + k) * HW + i), y);
    }
}

// Alg. 3 line 4-5: e = x̂ − t, c = 2σ² / (σ² + e²)² per pixel (K = 1).
__global__ void k_gm_weight(const float* __restrict__ x, const float* __restrict__ t, int64_t N, float s2,
                            float* __restrict__ c) {
    pdl_entry();
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < N; p += (int64_t)gridDim.x * blockDim.x) {
        const float e = x[p] - t[p];
        const float d = s2 + e * e;
        c[p] = 2.f * s2 / (d * d);
    }
}

// planar [K][stride] → canonical [M][K]; M = *Mdev (device count) when Mdev, else Mh
__global__ void k_export_vk(const float* __restrict__ src, const int* __restrict__ Mdev, int64_t Mh, int64_t stride,
                            int K, float* __restrict__ dst) {
    pdl_entry();
    const int64_t M = Mdev ? (int64_t)*Mdev : Mh;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * K; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i / K;
        const int k = (int)(i - v * K);
        dst[i] = src[(size_t)k * stride + v];
    }
}

// canonical [M][K] → planar [K][stride], optionally masked to live vertices (mu0 > 0)
__global__ void k_import_vk(const float* __restrict__ src, const float* __restrict__ mask, int64_t M, int64_t stride,
                            int K, float* __restrict__ dst) {
    pdl_entry();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * K; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i / K;
        const int k = (int)(i - v * K);
        dst[(size_t)k * stride + v] = (mask && !(mask[v] > 0.f)) ? 0.f : src[i];
    }
}

// Backward finalisation:  ∂t_k = c ∘ Sᵀd_k;
// ∂c = Σ_k Sᵀ(−d_k∘ŷ_k) + (Sᵀd_k)∘t_k   (reading #15).
__global__ void k_bwd_finalize(const int* __restrict__ vid, const float* __restrict__ db,
                               const float* __restrict__ y, const float* __restrict__ c, const float* __restrict__ t,
                               int64_t M, int K, int F, int64_t HW, float* __restrict__ dt, float* __restrict__ dc) {
    pdl_entry();
    const int64_t N = (int64_t)F * HW;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < N; p += (int64_t)gridDim.x * blockDim.x) {
        const int v = vid[p];
        const int f = (int)(p / HW);
        const int64_t pp = p - (int64_t)f * HW;
        const float cp = c[p];
        float acc = 0.f;
        for (int k = 0; k < K; ++k) {
            const float D = db[(size_t)k * M + v];
            const float Y = y[(size_t)k * M + v];
            const size_t ip = ((size_t)f * K + k) * HW + pp;
            dt[ip] = cp * D;
            acc += -D * Y + D * t[ip];
        }
        dc[p] = acc;
    }
}

// B̄ v (reading #4), debug / parity operator.
__global__ void k_blur(const int4* __restrict__ nbr, const float* __restrict__ x,
                       int64_t M, float bdiag, float* __restrict__ out) {
    pdl_entry();
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < M; v += (int64_t)gridDim.x * blockDim.x)
        out[v] = bdiag * x[v] + nbr_sum(x, (int)v, nbr[v]);
}

// A y for planar y (stride a.M), written canonical [M][K], M = the grid's vertex count (debug /
// parity operator).
__global__ void k_apply_A(VecArgs a, const float* __restrict__ ys, float* __restrict__ out) {
    pdl_entry();
    const int64_t M = a.frameOff[a.nf];
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < M; v += (int64_t)gridDim.x * blockDim.x)
        for (int k = 0; k < a.K; ++k)
            out[(size_t)v * a.K + k] =
                apply_A_row(ys + (size_t)k * a.M, a.n, (int)v, a.nbr[v], a.lam, a.sc[v]);
}

// M⁻¹ r at level 0 for masked planar w, written canonical [M][K] (debug / parity operator).
__global__ void k_precond_out(const float* __restrict__ w0, const float* __restrict__ mu0,
                              const int* __restrict__ parent0, const float* __restrict__ acc1, int64_t M1,
                              int64_t M, int64_t stride, int K, float* __restrict__ out) {
    pdl_entry();
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < M; v += (int64_t)gridDim.x * blockDim.x) {
        for (int k = 0; k < K; ++k) {
            float s = 0.f;
            if (mu0[v] > 0.f) {
                s = mu0[v] * w0[(size_t)k * stride + v];
                if (acc1) s += acc1[(size_t)k * M1 + parent0[v]];
            }
            out[(size_t)v * K + k] = s;
        }
    }
}

}  // namespace fbs
