// fbs_common.cuh — shared device helpers and handle layouts of the sm_100a bilateral solver.
// Unity build: api.cu includes every *.cuh of this directory.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <climits>

#include <atomic>
#include <cuda/atomic>
#include <vector>

#include "fbs.h"

namespace fbs {

// The device buffers of a handle (or of one call's scratch) and the allocator they come from:
// the process allocator current when the list is created (api.cu fbs_set_allocator); alloc ==
// nullptr means cudaMallocAsync / cudaFreeAsync.
fbs_allocator current_allocator();
struct AllocList {
    std::vector<void*> ptrs;
    fbs_allocator al = current_allocator();
    // arena (api.cu arena_reserve): later allocations are carved from it without a stream
    // operation, so the kernels enqueued between them keep their programmatic (PDL) chaining
    char* arena = nullptr;
    size_t arenaLeft = 0;
};

// a block of mapped pinned host memory from the staging pool (api.cu pinned_get / pinned_put)
struct PinnedBlock {
    void* p = nullptr;
    size_t bytes = 0;
    cudaEvent_t done = nullptr;
};

constexpr int kD = 5;                // XYLUV dims
constexpr int kCellMaxPx = 64;       // level-0 cell = one warp, ≤ 2 px per lane
constexpr int kCellsPerBlock = 8;    // 8 warps, one cell each
constexpr int kCoarseCap = 512;      // children of one pyramid coarse cell sorted in shared memory (larger: global scratch)
constexpr int kMaxLevels = 24;
#ifndef FBS_KTHREADS
#define FBS_KTHREADS 256
#endif
constexpr int kThreads = FBS_KTHREADS;  // vertex-parallel kernels
constexpr int kMaxK = 64;
constexpr int kVecPad = 512;         // vertex arrays streamed by bulk copies are allocated with this slack
constexpr int kScanTile = 256;       // tree-ordered level-1 positions per prefix-scan tile (tree_kernels.cuh)

// ------------------------------------------------------------------ launch counter
extern std::atomic<long long> g_launches;

// ------------------------------------------------------------------ programmatic dependent launch
// Every kernel is launched with programmatic stream serialization (api.cu launch_pdl) and starts
// here: it waits until the previous grid has completed and its memory is visible.  Data
// dependencies stay fully serial; what overlaps is the next kernel's launch processing and block
// dispatch with this grid's tail.  The dependent launch is triggered implicitly as this grid's
// blocks exit: an explicit griddepcontrol.launch_dependents at kernel entry (round 1's choice)
// let the next kernel's blocks claim SM slots while this one still needed them — measured 4.926
// vs 4.952 ms per bench step, configs[2] 1.14 vs 1.23 ms, configs[0] 0.86–0.89 vs 0.94 ms.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_entry() { pdl_wait(); }

// ------------------------------------------------------------------ bulk async copies (TMA engine)
// 1-D cp.async.bulk global → shared with mbarrier completion (sm_90+): one elected thread arms
// the barrier with the byte count and issues the copies; consumers wait on the phase parity.
// Addresses and sizes must be multiples of 16 bytes.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// The same copy with an L2 eviction-priority hint (a createpolicy cache policy): streamed-once
// operands evict first, so the data re-read by the next pass stays L2-resident.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// ------------------------------------------------------------------ small device helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic block sum (fixed tree).  All threads call; result valid in thread 0.
// `sh` needs blockDim.x/32 doubles.  Contains __syncthreads.
__device__ __forceinline__ double block_sum(double v, double* sh) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double r = 0.0;
    if (w == 0) {
        r = (l < (int)(blockDim.x >> 5)) ? sh[l] : 0.0;
        r = warp_sum(r);
    }
    return r;
}

// Two deterministic block sums in one pass (one barrier pair instead of two); the same fixed
// trees as block_sum, so each result is bitwise block_sum's.  `sh` needs 2·blockDim.x/32 ≤ 32
// doubles.  All threads call; results valid in thread 0.
__device__ __forceinline__ void block_sum2(double& v0, double& v1, double* sh) {
    v0 = warp_sum(v0);
    v1 = warp_sum(v1);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = (int)(blockDim.x >> 5);
    __syncthreads();
    if (l == 0) {
        sh[w] = v0;
        sh[16 + w] = v1;
    }
    __syncthreads();
    double r0 = 0.0, r1 = 0.0;
    if (w == 0) {
        r0 = (l < nw) ? sh[l] : 0.0;
        r1 = (l < nw) ? sh[16 + l] : 0.0;
        r0 = warp_sum(r0);
        r1 = warp_sum(r1);
    }
    v0 = r0;
    v1 = r1;
}

// Per-frame "last block done": every block of frame f calls this once after writing its
// partials; returns true (in all threads) only in the last block to arrive, which then owns
// the frame's final fixed-order reduction.  Resets the counter for the next launch.
// One fence per block, by the thread that signals (the grid-barrier pattern): the block barrier
// orders every thread's partial writes before thread 0's release fence, which is cumulative; the
// acquire fence before the second barrier covers the last block's reads.  Fencing in every
// thread made each wait for its own streaming stores (the SpMV's q) to be acknowledged.
__device__ __forceinline__ bool last_block_of_frame(unsigned* counter, int bpf, int* sflag) {
#ifdef FBS_FENCE_ALL
    __threadfence();
#endif
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned prev = atomicAdd(counter, 1u);
        const bool last = (prev == (unsigned)(bpf - 1));
        if (last) {
            __threadfence();
            *counter = 0u;
        }
        *sflag = last;
    }
    __syncthreads();
    return *sflag != 0;
}

// The same handshake when everything the last block reads was written by thread 0 itself (the
// block-reduced partials of write_partials / block_sum): no barrier before the signal, thread 0
// fences its own writes; one barrier broadcasts the outcome.
__device__ __forceinline__ bool last_block_t0(unsigned* counter, int bpf, int* sflag) {
    if (threadIdx.x == 0) {
        __threadfence();
        const bool last = atomicAdd(counter, 1u) == (unsigned)(bpf - 1);
        if (last) {
            __threadfence();
            *counter = 0u;
        }
        *sflag = last;
    }
    __syncthreads();
    return *sflag != 0;
}

// ------------------------------------------------------------------ decoupled look-back scan
// Tile state word: bits 63..62 flag (0 none, 1 aggregate, 2 inclusive prefix),
// bits 61..31 second count (pyramid children), bits 30..0 first count (vertices).
constexpr unsigned long long kLbAgg = 1ull << 62;
constexpr unsigned long long kLbPre = 2ull << 62;
constexpr unsigned long long kLbVal = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long lb_pack(unsigned a, unsigned b) {
    return (unsigned long long)a | ((unsigned long long)b << 31);
}
__device__ __forceinline__ unsigned lb_first(unsigned long long v) { return (unsigned)(v & 0x7fffffffull); }
__device__ __forceinline__ unsigned lb_second(unsigned long long v) {
    return (unsigned)((v >> 31) & 0x7fffffffull);
}

// Single-thread look-back (thread 0 of the tile).  Tiles obtain their id from an atomic
// counter, so every predecessor has already started: the spin is deadlock-free.
// Returns the exclusive prefix (packed) of tile `t`.
__device__ __forceinline__ unsigned long long lookback(unsigned long long* state, unsigned t,
                                                       unsigned long long agg) {
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> me(state[t]);
    if (t == 0) {
        me.store(kLbPre | agg, cuda::memory_order_relaxed);
        return 0ull;
    }
    me.store(kLbAgg | agg, cuda::memory_order_relaxed);
    unsigned long long excl = 0ull;
    long long j = (long long)t - 1;
    while (true) {
        cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> a(state[j]);
        const unsigned long long s = a.load(cuda::memory_order_relaxed);
        const unsigned long long fl = s & ~kLbVal;
        if (fl == 0ull) {
            __nanosleep(32);
            continue;
        }
        excl += s & kLbVal;
        if (fl == kLbPre) break;
        --j;
    }
    me.store(kLbPre | (excl + agg), cuda::memory_order_relaxed);
    return excl;
}


// Warp-parallel look-back (all 32 lanes of one warp call it): each round inspects the 32 closest
// predecessors at once, so the serial chain is ~window/32 loads instead of ~window.
__device__ __forceinline__ unsigned long long lookback_warp(unsigned long long* state, unsigned t,
                                                            unsigned long long agg) {
    const int lane = threadIdx.x & 31;
    if (lane == 0) {
        cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> me(state[t]);
        me.store((t == 0 ? kLbPre : kLbAgg) | agg, cuda::memory_order_relaxed);
    }
    if (t == 0) return 0ull;
    unsigned long long excl = 0ull;
    long long base = (long long)t - 1;
    while (true) {
        const long long j = base - lane;
        unsigned long long s = kLbPre;  // before tile 0: an inclusive prefix of 0
        if (j >= 0) {
            cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> a(state[j]);
            s = a.load(cuda::memory_order_relaxed);
            while ((s & ~kLbVal) == 0ull) {
                __nanosleep(20);
                s = a.load(cuda::memory_order_relaxed);
            }
        }
        const unsigned pre = __ballot_sync(0xffffffffu, (s & ~kLbVal) == kLbPre);
        const int stop = pre ? (__ffs(pre) - 1) : 31;  // closest predecessor with an inclusive prefix
        unsigned long long v = (lane <= stop) ? (s & kLbVal) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (pre) break;
        base -= 32;
    }
    if (lane == 0) {
        cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> me(state[t]);
        me.store(kLbPre | (excl + agg), cuda::memory_order_relaxed);
    }
    return excl;
}

// ------------------------------------------------------------------ neighbour encoding
// near: 8 signed bytes = relative offsets of the (x−, x+, l−, l+, u−, u+, v−, v+) neighbours
// (0 = absent; |offset| ≤ 127 because a σxy cell holds ≤ 64 vertices and x-neighbours sit in
// the adjacent cell of the same canonical row).  yoff: relative offsets of (y−, y+), 0 = absent.
// One int4 per vertex (16 B, a single 128-bit load): .x/.y = the 8 near offsets, .z/.w = y−, y+.
__device__ __forceinline__ int near_off(int4 nb, int i) {
    const unsigned w = (unsigned)((i < 4) ? nb.x : nb.y);
    return (int)(int8_t)(w >> (8 * (i & 3)));
}

// Σ_{u ∈ N(v)} x[u] in fixed slot order (x−,x+,l−,l+,u−,u+,v−,v+,y−,y+).
__device__ __forceinline__ float nbr_sum(const float* __restrict__ x, int v, int4 nb) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int o = near_off(nb, i);
        if (o) s += __ldg(x + v + o);
    }
    if (nb.z) s += __ldg(x + v + nb.z);
    if (nb.w) s += __ldg(x + v + nb.w);
    return s;
}

__device__ __forceinline__ bool is_isolated(int4 nb) { return (nb.x | nb.y | nb.z | nb.w) == 0; }

// ------------------------------------------------------------------ handles
struct Level {          // pyramid level k ≥ 1
    int64_t M = 0;      // vertices (all frames)
    int ncx = 0, ncy = 0;
    int64_t ncells = 0;
    uint64_t* keys = nullptr;       // [M]
    int* cellOff = nullptr;         // [ncells + 1]
    int* parent = nullptr;          // [M_{k-1}]  level k-1 → k  (S_{k-1})
    int* childStart = nullptr;      // [M + 1]
    int* childList = nullptr;       // [M_{k-1}]  children grouped by parent, fixed order
    int* count = nullptr;           // [M] P(1)
    int* cnt1 = nullptr;            // [M] level-1 descendants (k ≥ 2)
    std::vector<int64_t> frameOff;  // host copy [F + 1]
};

struct PcgScalars {     // per (frame, channel), fk = f*K + k
    double* rho = nullptr;
    double* alpha = nullptr;
    double* xalpha = nullptr; // hierarchical PCG: α of the x update (Alg. 2 line 8) the next direction
                              // pass applies (0: none); set by the SpMV's finish for every channel
    double* beta = nullptr;
    double* bb = nullptr;   // ‖b‖²
    double* rr = nullptr;   // last ‖r‖² (TOL)
    int* active = nullptr;
    int* iters = nullptr;
    int* status = nullptr;
    int* n_active = nullptr;  // single counter
};

// ------------------------------------------------------------------ hierarchy (tree_kernels.cuh)
struct HLevel {
    const int* parent = nullptr;      // level k → k+1 (canonical ids; nullptr at the top level)
    const int* childStart = nullptr;  // k ≥ 1: children (level k−1) of level-k vertices
    const int* childList = nullptr;
    const int* count = nullptr;       // k ≥ 1: P(1)
    const float* mu = nullptr;        // k ≥ 2: preconditioner multiplier (level 1: HierArgs::mu1T)
    const int2* rng = nullptr;        // k ≥ 2: (first tree position, count) of the level-1 descendants
    int64_t M = 0;
};

struct HierArgs {
    HLevel lv[kMaxLevels];
    int nt;                 // scan tiles of this launch (a frame group's HierArgs has its per-frame
                            // and per-tile pointers shifted to the group, api.cu)
    int L;                  // levels incl. base (max over frames)
    int F;
    int f0;                 // first frame of this launch's frame group (tileFrame holds global frames)
    int C;                  // channels carried through the pyramid
    const int* frameLevels;
    const int* lvFrameOff;  // [L][F+1] per-level frame vertex offsets (tree order keeps frames)
    double alpha, beta;     // z_weight parameters of the current use
    double zw[kMaxLevels];  // z_w(k) = α^−(β+k), k ≥ 1
    // tree order (grid)
    const int* tord0;       // [M0] level-0 vertex at each level-0 tree position
    const int2* ancRng;     // [top−2][M2] level-1 ranges of the level-k ancestors (k = 3..top) of level-2 vertices
    const float* ancMult;   // [top−2][M2] their multipliers of the current use (k_tree_anc_mult)
    const int* csT;         // [M1+1] level-0 tree range of the level-1 vertex at tree position i
    const int* parent0T;    // [M0] tree position of the level-1 parent of level-0 vertex v
    const int* tileFrameOff;  // [F+1] first scan tile of each frame
    const int* tileFrame;     // [nTiles1] frame of each scan tile
    const int2* tileRange;    // [nTiles1] tree positions [i0, i1) of each scan tile
    int nTiles1;
    int64_t M0, M1, M2;
    // per use (system buffers)
    float* mu1T;            // [M1] μ_1 in tree order
    float* buf1T;           // [C][M1] (P y)_1 in tree order
    double* locT;           // [C][M1] inclusive prefix within the scan tile
    double* tileAgg;        // [C][nTiles1] tile totals
    double* tileBase;       // [C][nTiles1] exclusive prefix of the tile totals within each frame
    unsigned* tcount;       // [C][F] tiles of each (frame, channel) lifted so far (k_tree_lift)
    int nfG;                // frames of this launch's group
    int coarseTiles;        // frames with more tiles get their tile bases from the lift (≤ kCoarseTiles)
    float* acc1T;           // [C][M1] projection of levels ≥ 1 onto level 1, tree order
    double* partial2;       // [F][bpf2][C] ρ partials of levels ≥ 1
    unsigned* counters;     // [F] last-block counters of the level-≥1 reductions
    int bpf2;               // blocks per frame of k_tree_coarse
};

// tree order of the pyramid (grid build)
struct TreeOrder {
    int* tord0 = nullptr;
    int* ancId = nullptr;    // [top−2][M2]
    int2* ancRng = nullptr;  // [top−2][M2]
    int* csT = nullptr;
    int* tord1 = nullptr;
    int* parent0T = nullptr;
    int* tileFrameOff = nullptr;
    int* tileFrame = nullptr;
    int2* tileRange = nullptr;
    int nTiles1 = 0;  // capacity of the tile arrays (the count is tileFrameOff[F] on the device)
    int2* rng[kMaxLevels] = {};
};

}  // namespace fbs

struct fbs_grid_s {
    int F = 0, H = 0, W = 0;
    std::vector<fbs::PinnedBlock> uploads;  // mapped pinned staging of the grid's small uploads
    double sxy = 0, sl = 0, suv = 0;
    int ncx = 0, ncy = 0;
    int64_t ncells = 0, N = 0, M = 0;  // M: level-0 vertex CAPACITY (= N; stride of vertex vectors)
    int n_bistoch = 20;
    int dims = 5;               // D (5: XYLUV; 3: XYL of a grayscale reference)
    bool has_pyramid = false;
    cudaStream_t stream = nullptr;
    int device = 0;
    // level 0
    int* colStart = nullptr;   // [ncx + 1]
    int* rowStart = nullptr;   // [ncy + 1]
    int* vid = nullptr;        // [N]
    uint64_t* keys = nullptr;  // [N] capacity (first M valid)
    int* m = nullptr;          // [N] capacity
    int* cellOff = nullptr;    // [ncells + 1]
    uint8_t* perm = nullptr;   // [ncells][64] sorted position → the pixel's row·8 + column in its cell
    unsigned long long* heads = nullptr;  // [ncells] run-head bits of the sorted positions (vertex ranks)
    int4* nbr = nullptr;       // [M] packed neighbour offsets (fbs_common.cuh near_off)
    float* n = nullptr;        // [M]
    int* frameOff = nullptr;   // device [F + 1]
    std::vector<int64_t> frameOffH;
    int* frameLevels = nullptr;  // device [F]
    std::vector<int> frameLevelsH;
    float bistoch_residual = -1.f;
    int L = 1;  // levels carried by the hierarchy kernels (Lmax: an upper bound of every frame's)
    int* err = nullptr;             // device: build invariant flags (checked by ensure_sizes)
    std::vector<int64_t> capH;      // capacity of each level (level 0: N)
    // exact sizes, read back on demand by the synchronous query/export calls (api.cu ensure_sizes)
    bool sized = false;
    int64_t Mx = 0;                 // level-0 vertices
    int Lx = 1;                     // levels incl. base (max over frames)
    std::vector<int64_t> levelMx;   // vertices of each level (all frames)
    fbs::Level lv[fbs::kMaxLevels];
    int64_t maxFrameM = 0;
    int64_t maxFrameM1 = 0;
    int64_t maxFrameM2 = 0;
    int* lvFrameOffDev = nullptr;  // [L][F + 1]
    fbs::TreeOrder tree;           // tree order of the pyramid (L > 1)
    fbs::AllocList allocs;
};

struct fbs_system_s {
    fbs_grid g = nullptr;
    int K = 1;
    double lam = 1.0;
    fbs_solve_opts o{};
    cudaStream_t stream = nullptr;
    cudaStream_t capture = nullptr;
    int BPF = 1;
    int BPFs = 1;             // blocks per (frame, channel) of the channel-split kernels (K > 1)
    int BPFl0 = 1;            // blocks per frame of the PCG direction kernel (k_tree_level0<PCG>)
    int BPFk = 1;             // blocks per frame of the channel-joint SpMV (k_spmv_kjoint, K > 1)
    int* inflags = nullptr;   // input-check status bits (FBS_ST_NEG_CONF, FBS_ST_NONFINITE)
    int nGroups = 2;          // frame groups of the FIXED-mode PCG (run_pcg); FBS_PCG_GROUPS=1 disables
    // vertex arrays
    float* sc = nullptr;      // [M]
    float* b = nullptr;       // [K][M] S(c∘t)
    float* u = nullptr;       // [K][M] S g (backward right-hand side)
    float* diagA = nullptr;   // [M] Laplacian-form diag(A); 0 ⇔ dead vertex
    float* mu0 = nullptr;     // [M] level-0 multiplier (1/diagA on live vertices)
    float* y0 = nullptr;      // [K][M] initial state
    float* xh = nullptr;      // [K][M] forward solution ŷ
    float* xb = nullptr;      // [K][M] backward solution ∂f/∂b
    float* rh = nullptr;
    float2* dn = nullptr;     // [K][M] interleaved (d, n)
    float* qh = nullptr;
    float* sh = nullptr;
    float* w0 = nullptr;                   // [C][M] level-0 pyramid input (init, μ_k, debug operator)
    float* mu[fbs::kMaxLevels] = {};       // [M_k] precond multipliers (k ≥ 2 canonical; k = 1 tree order)
    float* ancMult = nullptr;              // [top−2][M2] multipliers of the level-2 vertices' ancestors
    float* buf1T = nullptr;                // [C][M1] hierarchy work arrays (tree_kernels.cuh)
    double* locT = nullptr;
    double* tileAgg = nullptr;
    double* tileBase = nullptr;
    unsigned* tcount = nullptr;
    float* acc1T = nullptr;
    double* partial2 = nullptr;
    int bpf2 = 1;
    int bpf2g = 0;            // > 0: the PCG coarse pass runs 8 lanes per level-2 vertex with these blocks per frame
    int C = 1;
    double* partial = nullptr;  // [F][BPF][2K]
    unsigned* counters = nullptr;  // [F][K] (VecArgs kernels)
    unsigned* counters2 = nullptr; // [F] (HierArgs kernels)
    fbs::PcgScalars fwd, bwd;
    bool useHierP = false;
    // r is 0 on dead vertices (b = S(c∘t) is, and A's rows are 0 there), so w = mask∘r = r and the
    // lift reads r instead of a materialised w (forward solves); the backward's u = S g is not
    bool rMasked = false;
    fbs::HierArgs hP{};
    bool has_backward = false;
    int* lr_rank = nullptr;    // low-rank solves: kept rank t_f per frame (device)
    fbs::AllocList allocs;
};
