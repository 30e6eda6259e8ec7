// lowrank_kernels.cuh — low-rank reduction of the multi-channel right-hand sides (Supp. §4,
// PAPER.md:867-900): B P = Q R, keep the rows of R' = sort(R Pᵀ) carrying ≥ (1 − ε) of the
// mass (reading #26), solve A Ỹ = Q̃ and expand Y = Ỹ R̃.
//
// On the GPU the pivoted QR of the tall, thin B_f = [b_0 … b_{K−1}] (one per frame) is taken
// through its Gram matrix: G = B_fᵀ B_f in fp64, then a pivoted Cholesky G = (R P)ᵀ(R P) with
// the pivot rule of column-pivoted QR (largest remaining column norm; ties → lowest index).
// In exact arithmetic this R equals the QR's R up to row signs, so R̃ and Q̃ R̃ are the same;
// Q̃ = B_f T with T = P R⁻¹ restricted to the kept rows.  K ≤ 64.
#pragma once
#include "fbs_common.cuh"
#include "solve_kernels.cuh"

namespace fbs {

constexpr int kGramTile = 64;  // vertices staged per round

// Per-frame blocks (bpf per frame): partial Gram sums over the block's vertices, pair p = (k ≤ l)
// in row-major upper-triangle order; the last block of the frame adds the partials in a fixed
// order → G [F][K][K] (fp64, symmetric, both halves written).
__global__ void __launch_bounds__(256) k_gram(const float* __restrict__ b, int64_t M, int K, const int* __restrict__ frameOff,
                                              int bpf, double* __restrict__ partial, unsigned* __restrict__ counters,
                                              double* __restrict__ G) {
    pdl_entry();
    __shared__ float tile[kMaxK][kGramTile];
    __shared__ int sflag;
    const int f = blockIdx.x / bpf, j = blockIdx.x % bpf;
    const int v0 = frameOff[f], v1 = frameOff[f + 1];
    const int P = K * (K + 1) / 2;
    constexpr int kPairsPerThread = (kMaxK * (kMaxK + 1) / 2 + 255) / 256;
    double acc[kPairsPerThread];
    int pk[kPairsPerThread], pl[kPairsPerThread];
#pragma unroll
    for (int q = 0; q < kPairsPerThread; ++q) {
        acc[q] = 0.0;
        int p = threadIdx.x + 256 * q, k = 0;
        pk[q] = -1;
        pl[q] = -1;
        if (p < P) {  // p → (k, l), k ≤ l
            while (p >= K - k) {
                p -= K - k;
                ++k;
            }
            pk[q] = k;
            pl[q] = k + p;
        }
    }
    for (int vb = v0 + j * kGramTile; vb < v1; vb += bpf * kGramTile) {
        const int n = min(kGramTile, v1 - vb);
        for (int i = threadIdx.x; i < K * kGramTile; i += blockDim.x) {
            const int k = i / kGramTile, u = i % kGramTile;
            tile[k][u] = (u < n) ? b[(size_t)k * M + vb + u] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kPairsPerThread; ++q) {
            if (pk[q] < 0) continue;
            double s = 0.0;
            for (int u = 0; u < n; ++u) s += (double)tile[pk[q]][u] * (double)tile[pl[q]][u];
            acc[q] += s;
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < kPairsPerThread; ++q) {
        const int p = threadIdx.x + 256 * q;
        if (p < P) partial[((size_t)f * bpf + j) * P + p] = acc[q];
    }
    if (last_block_of_frame(counters + f, bpf, &sflag)) {
#pragma unroll
        for (int q = 0; q < kPairsPerThread; ++q) {
            if (pk[q] < 0) continue;
            const int p = threadIdx.x + 256 * q;
            double s = 0.0;
            for (int jj = 0; jj < bpf; ++jj) s += __ldcg(partial + ((size_t)f * bpf + jj) * P + p);
            G[((size_t)f * K + pk[q]) * K + pl[q]] = s;
            G[((size_t)f * K + pl[q]) * K + pk[q]] = s;
        }
    }
}

// One block per frame: pivoted Cholesky of G_f, row masses of R Pᵀ, mass-sorted rows, the kept
// count t_f, the expansion rows Rt_f [K][K] (row a = kept row a of R Pᵀ, zero beyond t_f) and the
// reduction T_f [K][K] (column a = P R⁻¹ column of kept row a, zero beyond t_f).
__global__ void __launch_bounds__(64) k_pchol(const double* __restrict__ G, int K, double eps, int* __restrict__ tOut,
                                              double* __restrict__ Rt, double* __restrict__ T) {
    pdl_entry();
    __shared__ double R[kMaxK][kMaxK + 1];   // R[row][position]
    __shared__ double d[kMaxK];              // remaining diagonal, by original column
    __shared__ double mass[kMaxK];
    __shared__ int perm[kMaxK], order[kMaxK];
    __shared__ int s_rank, s_t;
    const int f = blockIdx.x;
    const double* Gf = G + (size_t)f * K * K;
    for (int i = threadIdx.x; i < kMaxK * (kMaxK + 1); i += blockDim.x) R[i / (kMaxK + 1)][i % (kMaxK + 1)] = 0.0;
    __syncthreads();
    for (int i = threadIdx.x; i < K; i += blockDim.x) {
        perm[i] = i;
        d[i] = Gf[(size_t)i * K + i];
    }
    if (threadIdx.x == 0) s_rank = K;
    __syncthreads();
    for (int j = 0; j < K; ++j) {
        if (threadIdx.x == 0) {  // pivot: largest remaining norm, ties → lowest position
            int p = j;
            for (int i = j + 1; i < K; ++i)
                if (d[perm[i]] > d[perm[p]]) p = i;
            if (p != j) {
                const int tmp = perm[j];
                perm[j] = perm[p];
                perm[p] = tmp;
                for (int q = 0; q < j; ++q) {
                    const double r = R[q][j];
                    R[q][j] = R[q][p];
                    R[q][p] = r;
                }
            }
            const double dp = d[perm[j]];
            if (!(dp > 0.0)) s_rank = j;
            else R[j][j] = sqrt(dp);
        }
        __syncthreads();
        if (s_rank <= j) break;
        const int pj = perm[j];
        for (int i = j + 1 + threadIdx.x; i < K; i += blockDim.x) {
            double s = Gf[(size_t)pj * K + perm[i]];
            for (int q = 0; q < j; ++q) s -= R[q][j] * R[q][i];
            const double r = s / R[j][j];
            R[j][i] = r;
            d[perm[i]] -= r * r;
        }
        __syncthreads();
    }
    // masses of the rows of R Pᵀ (= of R), mass-sorted order (stable), kept count
    for (int r = threadIdx.x; r < K; r += blockDim.x) {
        double m = 0.0;
        for (int i = 0; i < K; ++i) m += R[r][i] * R[r][i];
        mass[r] = m;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 0; i < K; ++i) order[i] = i;
        for (int i = 1; i < K; ++i) {  // insertion sort, descending, stable
            const int o = order[i];
            int q = i - 1;
            while (q >= 0 && mass[order[q]] < mass[o]) {
                order[q + 1] = order[q];
                --q;
            }
            order[q + 1] = o;
        }
        double total = 0.0;
        for (int i = 0; i < K; ++i) total += mass[i];
        int t = 0;
        if (total > 0.0) {
            double cum = 0.0;
            t = K;
            for (int i = 0; i < K; ++i) {
                cum += mass[order[i]];
                if (cum >= (1.0 - eps) * total - 1e-12 * total) {
                    t = i + 1;
                    break;
                }
            }
            t = min(t, s_rank);
        }
        s_t = t;
        tOut[f] = t;
    }
    __syncthreads();
    double* Rtf = Rt + (size_t)f * K * K;
    double* Tf = T + (size_t)f * K * K;
    for (int i = threadIdx.x; i < K * K; i += blockDim.x) {
        Rtf[i] = 0.0;
        Tf[i] = 0.0;
    }
    __syncthreads();
    // kept row a = R row order[a]: Rt[a][perm[i]] = R[order[a]][i]; T[:, a] = P R⁻¹[:, order[a]]
    for (int a = threadIdx.x; a < s_t; a += blockDim.x) {
        const int jr = order[a];
        for (int i = 0; i < K; ++i) Rtf[(size_t)a * K + perm[i]] = R[jr][i];
        double x[kMaxK];
        for (int i = 0; i < kMaxK; ++i) x[i] = 0.0;
        x[jr] = 1.0 / R[jr][jr];  // back substitution for column jr of R⁻¹
        for (int i = jr - 1; i >= 0; --i) {
            double s = 0.0;
            for (int q = i + 1; q <= jr; ++q) s += R[i][q] * x[q];
            x[i] = -s / R[i][i];
        }
        for (int i = 0; i <= jr; ++i) Tf[(size_t)perm[i] * K + a] = x[i];
    }
}

// b'[a][v] = Σ_k b[k][v] T_f[k][a]  (Q̃ columns, a < Kc; per-frame blocks)
__global__ void k_reduce_rhs(const float* __restrict__ b, int64_t M, int K, int Kc, const int* __restrict__ frameOff,
                             int bpf, const double* __restrict__ T, float* __restrict__ bout) {
    pdl_entry();
    const int f = blockIdx.x / bpf, j = blockIdx.x % bpf;
    const double* Tf = T + (size_t)f * K * K;
    for (int v = frameOff[f] + j * blockDim.x + threadIdx.x; v < frameOff[f + 1]; v += bpf * blockDim.x) {
        float bv[kMaxK];
        for (int k = 0; k < K; ++k) bv[k] = b[(size_t)k * M + v];
        for (int a = 0; a < Kc; ++a) {
            double s = 0.0;
            for (int k = 0; k < K; ++k) s += (double)bv[k] * Tf[(size_t)k * K + a];
            bout[(size_t)a * M + v] = (float)s;
        }
    }
}

// y[k][v] = Σ_a ỹ[a][v] Rt_f[a][k]  (expansion Y = Ỹ R̃; per-frame blocks)
__global__ void k_expand(const float* __restrict__ yr, int64_t M, int K, int Kc, const int* __restrict__ frameOff,
                         int bpf, const double* __restrict__ Rt, float* __restrict__ y) {
    pdl_entry();
    const int f = blockIdx.x / bpf, j = blockIdx.x % bpf;
    const double* Rf = Rt + (size_t)f * K * K;
    for (int v = frameOff[f] + j * blockDim.x + threadIdx.x; v < frameOff[f + 1]; v += bpf * blockDim.x) {
        float yv[kMaxK];
        for (int a = 0; a < Kc; ++a) yv[a] = yr[(size_t)a * M + v];
        for (int k = 0; k < K; ++k) {
            double s = 0.0;
            for (int a = 0; a < Kc; ++a) s += (double)yv[a] * Rf[(size_t)a * K + k];
            y[(size_t)k * M + v] = (float)s;
        }
    }
}

}  // namespace fbs
