// api.cu — C ABI (include/fbs.h) and host orchestration of the sm_100a bilateral solver.
// Unity build: this translation unit includes every kernel header of csrc/.
#include <algorithm>
#include <cstdlib>
#include <utility>
#include <cmath>
#include <functional>
#include <map>
#include <chrono>
#include <cstdio>
#include <mutex>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>

#include "fbs_common.cuh"
#include "grid_kernels.cuh"
#include "pyramid_kernels.cuh"
#include "solve_kernels.cuh"
#include "tree_kernels.cuh"
#include "lowrank_kernels.cuh"
#include "dt_kernels.cuh"

namespace fbs {

std::atomic<long long> g_launches{0};

// the process allocator for handles created from now on (fbs_set_allocator)
std::mutex g_alloc_mu;
fbs_allocator g_allocator{};
fbs_allocator current_allocator() {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    return g_allocator;
}

namespace {

thread_local std::string t_err;

struct Err : std::runtime_error {
    int code;
    Err(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        const int code = (e == cudaErrorMemoryAllocation) ? FBS_ENOMEM : FBS_ECUDA;
        throw Err(code, std::string(what) + ": " + cudaGetErrorString(e));
    }
}

// PDL is used only between BACK-TO-BACK kernels of the library on a stream: after any other
// operation on the stream (allocation, free, copy, event record/wait, or the caller's work before
// an API call) the next launch is fully serialised.  A programmatic edge across an intervening
// stream operation is not ordered after the kernel before it (measured: a grid build with a
// stream-ordered allocation between two PDL kernels read stale data), so pdl_break marks the
// stream and launch_pdl consumes the mark.
thread_local std::vector<cudaStream_t> t_pdl_broken;
int pdl_break_mask() {  // DEBUG A/B: which operations break the PDL chain (bit 0 alloc, 1 free, 2 copy/event, 3 entry)
    static const int m = [] {
        const char* e = std::getenv("FBS_PDL_BREAK");
        return e ? std::atoi(e) : 63;
    }();
    return m;
}
void pdl_break(cudaStream_t s, int kind);
bool pdl_every_level() {  // DEBUG A/B: serialise every pyramid level, not only the first
    static const bool on = std::getenv("FBS_PDL_EVERY_LEVEL") != nullptr;
    return on;
}
void pdl_break(cudaStream_t s) { pdl_break(s, 4); }
void pdl_break(cudaStream_t s, int kind) {
    if (!(pdl_break_mask() & kind)) return;
    if (std::find(t_pdl_broken.begin(), t_pdl_broken.end(), s) == t_pdl_broken.end()) t_pdl_broken.push_back(s);
}
bool pdl_take(cudaStream_t s) {
    auto it = std::find(t_pdl_broken.begin(), t_pdl_broken.end(), s);
    if (it == t_pdl_broken.end()) return true;
    t_pdl_broken.erase(it);
    return false;
}
cudaError_t memcpy_async(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t s) {
    pdl_break(s);
    return cudaMemcpyAsync(dst, src, bytes, kind, s);
}
cudaError_t event_record(cudaEvent_t e, cudaStream_t s) {
    pdl_break(s);
    return cudaEventRecord(e, s);
}
cudaError_t stream_wait(cudaStream_t s, cudaEvent_t e) {
    pdl_break(s);
    return cudaStreamWaitEvent(s, e, 0);
}

// ---- per-kernel event timing (fbs_profile_*)
struct ProfRec {
    const char* name;
    cudaEvent_t a, b;
    cudaStream_t s;
};
std::atomic<int> g_prof_on{0};
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_ev_pool;
std::mutex g_prof_mu;

cudaEvent_t ev_get() {
    if (!g_ev_pool.empty()) {
        cudaEvent_t e = g_ev_pool.back();
        g_ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "cudaEventCreate");
    return e;
}

struct ProfScope {
    int idx = -1;
    cudaStream_t s;
    ProfScope(const char* name, cudaStream_t st) : s(st) {
        if (!g_prof_on.load(std::memory_order_relaxed)) return;
        std::lock_guard<std::mutex> lk(g_prof_mu);
        ProfRec r{name, ev_get(), ev_get(), st};
        ck(cudaEventRecord(r.a, s), "cudaEventRecord");  // timing events keep the PDL chain (as unprofiled)
        g_prof.push_back(r);
        idx = (int)g_prof.size() - 1;
    }
    ~ProfScope() {
        if (idx < 0) return;
        std::lock_guard<std::mutex> lk(g_prof_mu);
        cudaEventRecord(g_prof[idx].b, s);
    }
};

// Every launch uses programmatic stream serialization (fbs_common.cuh pdl_entry); FBS_NO_PDL=1
// in the environment turns it off (A/B measurement).
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FBS_NO_PDL");
        return !(e && e[0] == '1');
    }();
    return on;
}

// DEBUG: FBS_PDL_BREAK_BEFORE=name1,name2 serialises the launches of those kernels (bisecting
// PDL ordering problems)
void pdl_debug_break(const char* name, cudaStream_t s) {
    static const std::string list = [] {
        const char* e = std::getenv("FBS_PDL_BREAK_BEFORE");
        return e ? "," + std::string(e) + "," : std::string();
    }();
    if (!list.empty() && list.find("," + std::string(name) + ",") != std::string::npos) pdl_break(s, 16);
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (pdl_take(s) && pdl_enabled()) ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

#define LAUNCH(kernel, grid, block, smem, stream, ...) LAUNCH_AS(#kernel, kernel, grid, block, smem, stream, __VA_ARGS__)
#define LAUNCH_AS(name, kernel, grid, block, smem, stream, ...)                          \
    do {                                                                                 \
        ::fbs::pdl_debug_break((name), (stream));                                        \
        ::fbs::ProfScope _ps((name), (stream));                                          \
        ck(::fbs::launch_pdl(kernel, dim3(grid), dim3(block), (smem), (stream), __VA_ARGS__), #kernel); \
        ::fbs::g_launches.fetch_add(1, std::memory_order_relaxed);                       \
    } while (0)

int g_num_sms = 0;

void device_setup(int* dev) {
    ck(cudaGetDevice(dev), "cudaGetDevice");
    static bool pool_done[64] = {};
    if (*dev < 64 && !pool_done[*dev]) {
        cudaMemPool_t pool;
        ck(cudaDeviceGetDefaultMemPool(&pool, *dev), "cudaDeviceGetDefaultMemPool");
        uint64_t thr = UINT64_MAX;
        ck(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr), "mempool threshold");
        int sms = 0;
        ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, *dev), "sm count");
        g_num_sms = sms;
        ck(cudaFuncSetAttribute(k_bistoch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBsSmem), "k_bistoch smem");
        pool_done[*dev] = true;
    }
}

void* raw_alloc(AllocList& list, size_t bytes, cudaStream_t s) {
    pdl_break(s, 1);  // a stream-ordered allocation between PDL launches breaks their ordering
    void* p = nullptr;
    if (list.al.alloc) {
        p = list.al.alloc(bytes, list.al.ctx, reinterpret_cast<fbs_stream>(s));
        if (!p) throw Err(FBS_ENOMEM, "caller allocator returned NULL");
        // vector loads (int4 / float4) and cp.async.bulk copies need 16-byte-aligned buffers (fbs.h)
        if (reinterpret_cast<uintptr_t>(p) & 15) {
            list.al.free(p, list.al.ctx, reinterpret_cast<fbs_stream>(s));
            throw Err(FBS_EINVAL, "caller allocator returned a pointer that is not 16-byte aligned");
        }
    } else {
        ck(cudaMallocAsync(&p, bytes, s), "cudaMallocAsync");
    }
    list.ptrs.push_back(p);
    return p;
}

// One allocation up front for a handle's buffers (its size an estimate; dalloc falls back to
// separate allocations once it is used up).
void arena_reserve(AllocList& list, size_t bytes, cudaStream_t s) {
    bytes = (bytes + 255) & ~size_t(255);
    list.arena = static_cast<char*>(raw_alloc(list, bytes, s));
    list.arenaLeft = bytes;
}

template <class T>
T* dalloc(AllocList& list, size_t count, cudaStream_t s) {
    if (count == 0) count = 1;
    const size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);  // 256-byte aligned carving
    if (list.arena && bytes <= list.arenaLeft) {
        void* p = list.arena;
        list.arena += bytes;
        list.arenaLeft -= bytes;
        return static_cast<T*>(p);
    }
    return static_cast<T*>(raw_alloc(list, count * sizeof(T), s));
}
void free_all(AllocList& list, cudaStream_t s) {
    pdl_break(s, 2);
    for (void* p : list.ptrs) {
        if (list.al.free) list.al.free(p, list.al.ctx, reinterpret_cast<fbs_stream>(s));
        else cudaFreeAsync(p, s);
    }
    list.ptrs.clear();
}

// Side streams of the frame-group splits (Alg. 1 and the FIXED-mode PCG), created once per (device,
// caller stream).
cudaStream_t group_stream(int dev, cudaStream_t caller, int i) {
    // one set per (device, caller stream): solves issued on different caller streams stay
    // independent instead of serialising on shared side streams
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, std::vector<cudaStream_t>> streams;
    std::lock_guard<std::mutex> lk(mu);
    auto& v = streams[{dev, caller}];
    while ((int)v.size() <= i) {
        cudaStream_t st;
        ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
        v.push_back(st);
    }
    return v[i];
}

// ---- small host <-> device transfers through mapped pinned memory and a copy kernel.
// cudaMemcpyAsync queues on the copy engines behind whatever bulk copies other streams have in
// flight (a caller's 66 MB result read-back or 182 MB input upload), which stalled the grid
// build's level-size read-backs by up to a millisecond per step in a pipelined caller.  A kernel
// reading or writing mapped host memory (device address = host address under UVA) does not wait
// on the copy engines.  Buffers come from a process-wide pool; a returned buffer carries an event
// recorded on the stream of its last use and is reused only once that event has completed.
std::mutex g_pin_mu;
std::vector<PinnedBlock> g_pin_free;

PinnedBlock pinned_get(size_t bytes) {
    {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        for (size_t i = 0; i < g_pin_free.size(); ++i) {
            PinnedBlock b = g_pin_free[i];
            if (b.bytes >= bytes && (!b.done || cudaEventQuery(b.done) == cudaSuccess)) {
                g_pin_free.erase(g_pin_free.begin() + i);
                return b;
            }
        }
    }
    PinnedBlock b;
    b.bytes = std::max<size_t>(bytes, 64 * 1024);
    ck(cudaHostAlloc(&b.p, b.bytes, cudaHostAllocMapped | cudaHostAllocPortable), "cudaHostAlloc");
    ck(cudaEventCreateWithFlags(&b.done, cudaEventDisableTiming), "event");
    return b;
}

void pinned_put(PinnedBlock b, cudaStream_t s) {
    if (!b.p) return;
    event_record(b.done, s);
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_free.push_back(b);
}

__global__ void k_copy_words(const int* __restrict__ src, int* __restrict__ dst, int64_t n) {
    pdl_entry();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

__global__ void k_fill_words(int* __restrict__ dst, int64_t n, int value) {
    pdl_entry();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = value;
}

__global__ void k_zero_words(int* __restrict__ dst, int64_t n) {
    pdl_entry();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = 0;
}

// zero `bytes` (a multiple of 4) of device memory with a kernel (cudaMemsetAsync may queue on a copy
// engine behind a caller's bulk transfers)
void zero_words(void* dst, size_t bytes, cudaStream_t s) {
    const int64_t n = (int64_t)(bytes / 4);
    if (n == 0) return;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 1024);
    LAUNCH(k_zero_words, blocks, 256, 0, s, static_cast<int*>(dst), n);
}

// copy `bytes` (a multiple of 4) between device memory and a mapped pinned block, in stream order
void copy_words(const void* src, void* dst, size_t bytes, cudaStream_t s) {
    const int64_t n = (int64_t)(bytes / 4);
    if (n == 0) return;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 1024);
    LAUNCH(k_copy_words, blocks, 256, 0, s, static_cast<const int*>(src), static_cast<int*>(dst), n);
}

inline int grid_for(int64_t n, int threads = kThreads, int cap_per_sm = 16) {
    int64_t b = (n + threads - 1) / threads;
    const int64_t cap = (int64_t)(g_num_sms > 0 ? g_num_sms : 148) * cap_per_sm;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

int bitlen(int64_t v) {
    int b = 0;
    while (v > 0) {
        ++b;
        v >>= 1;
    }
    return b;
}

int guard(const char* where, const std::function<void()>& body);

}  // namespace
}  // namespace fbs

using namespace fbs;


// ===================================================================================== grid
// Pyramid levels carried (Lmax: halving until every coordinate is 0) and the vertex capacity of
// each level: a level-k vertex is a distinct (level-k cell, halved code) pair with at least one
// child, so M_k ≤ min(M_{k−1}, cells_k · codes_k); level 0: M ≤ N.
static std::vector<int64_t> level_caps(int F, int ncx, int ncy, int64_t N, double sl, double suv, int dims, bool pyr) {
    const int64_t lmax = (int64_t)std::floor(65280.0 / (256.0 * sl));
    const int64_t uvmax = (dims == 3) ? 0 : (int64_t)std::floor(65408.0 / (256.0 * suv));
    int Lmax = 1;
    if (pyr) {
        const int bits = std::max({bitlen(ncy - 1), bitlen(ncx - 1), bitlen(lmax), bitlen(uvmax)});
        Lmax = std::min(1 + bits, kMaxLevels);
    }
    std::vector<int64_t> cap(Lmax, N);
    for (int k = 1; k < Lmax; ++k) {
        const int64_t nck = (int64_t)F * (((ncx - 1) >> k) + 1) * (((ncy - 1) >> k) + 1);
        const double codes = (double)((lmax >> k) + 1) * (double)((uvmax >> k) + 1) * (double)((uvmax >> k) + 1);
        cap[k] = std::max<int64_t>(1, (int64_t)std::min<double>((double)cap[k - 1], (double)nck * codes));
    }
    return cap;
}

// Device bytes of a grid's buffers (the arena estimate; a shortfall only costs extra allocations)
static size_t grid_bytes(int F, int ncx, int ncy, int64_t N, int64_t ncells, const std::vector<int64_t>& cap) {
    const int L = (int)cap.size();
    size_t b = (size_t)N * (4 + 8 + 4 + 16 + 4 + 4) + (size_t)ncells * (kCellMaxPx + 4 + 4 + 8) + (size_t)8 * kVecPad * 16;
    if (L > 1) {
        b += (size_t)N * (16 + 4 + 4 + 4);  // pyramid scratch + ranks, tord0, parent0T
        for (int k = 1; k < L; ++k) {
            const int64_t nck = (int64_t)F * (((ncx - 1) >> k) + 1) * (((ncy - 1) >> k) + 1);
            b += (size_t)cap[k] * (8 + 4 + 4 + 4 + 8 + 8) + (size_t)cap[k - 1] * 8 + (size_t)nck * 8 + 4096;
        }
        b += (size_t)cap[1] * 8 + (size_t)(L > 3 ? L - 3 : 0) * (L > 2 ? cap[2] : 0) * 12;
        b += ((size_t)cap[1] / kScanTile + F + 1) * 12;
    }
    return b + ((size_t)L + 8) * (F + 1) * 4 + (1 << 20);
}

static void grid_build_impl(const uint8_t* rgb, int F, int H, int W, double sxy, double sl, double suv,
                            const fbs_grid_opts* opts, cudaStream_t s, fbs_grid* out) {
    if (!rgb || !out) throw Err(FBS_EINVAL, "null pointer");
    if (F < 1 || F > 256) throw Err(FBS_EINVAL, "frames must be in [1, 256]");
    if (!(sxy >= 1.0) || !(sl >= 1.0) || !(suv >= 1.0) || !std::isfinite(sxy) || !std::isfinite(sl) ||
        !std::isfinite(suv))
        throw Err(FBS_EINVAL, "sigma_xy, sigma_l, sigma_uv must be finite and >= 1");
    if (H < 1 || W < 1) throw Err(FBS_EINVAL, "height and width must be >= 1");
    const int ncx = (int)std::floor((double)(W - 1) / sxy) + 1;
    const int ncy = (int)std::floor((double)(H - 1) / sxy) + 1;
    if (ncx > 65536 || ncy > 65536) throw Err(FBS_EINVAL, "image too large for 16-bit spatial key fields");
    // widest cell: ⌈σxy⌉ columns at most; the kernel re-checks every cell
    const int cw = (int)std::ceil(sxy);
    if ((int64_t)std::min(cw, W) * std::min(cw, H) > kCellMaxPx)
        throw Err(FBS_EINVAL, "a sigma_xy cell would hold more than 64 pixels (sigma_xy > 8 is not supported)");
    const int64_t N = (int64_t)F * H * W;
    if (N >= (1ll << 31) - 1) throw Err(FBS_EINVAL, "too many pixels (>= 2^31)");

    int dev = 0;
    device_setup(&dev);
    pdl_break(s, 8);  // the caller's own work may precede this call on the stream
    // FBS_HOST_TIMING=1: host-side timestamps of the grid build (diagnostic)
    static const bool host_timing = std::getenv("FBS_HOST_TIMING") && std::getenv("FBS_HOST_TIMING")[0] == '1';
    auto t_prev = std::chrono::steady_clock::now();
    auto HT = [&](const char* what) {
        if (!host_timing) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[fbs host] %-28s %8.1f us\n", what,
                     std::chrono::duration<double, std::micro>(now - t_prev).count());
        t_prev = now;
    };
    fbs_grid g = new fbs_grid_s();
    bool pyrForked = false;  // work was enqueued on the pyramid's side stream
    try {
        g->F = F; g->H = H; g->W = W; g->sxy = sxy; g->sl = sl; g->suv = suv;
        g->ncx = ncx; g->ncy = ncy; g->ncells = (int64_t)F * ncx * ncy; g->N = N;
        g->n_bistoch = opts ? opts->n_bistoch : 20;
        g->dims = opts ? opts->dims : 5;
        if (g->dims != 5 && g->dims != 3) throw Err(FBS_EINVAL, "dims must be 5 or 3");
        if (g->n_bistoch < 0) throw Err(FBS_EINVAL, "n_bistoch must be >= 0");
        const bool want_pyr = opts ? opts->build_pyramid != 0 : true;
        g->stream = s;
        g->device = dev;
        auto& A = g->allocs;
        const std::vector<int64_t> cap = level_caps(F, ncx, ncy, N, sl, suv, g->dims, want_pyr);
        arena_reserve(A, grid_bytes(F, ncx, ncy, N, g->ncells, cap), s);

        g->colStart = dalloc<int>(A, ncx + 1, s);
        g->rowStart = dalloc<int>(A, ncy + 1, s);
        LAUNCH(k_axis_bins, grid_for(W), kThreads, 0, s, W, sxy, ncx, g->colStart);
        LAUNCH(k_axis_bins, grid_for(H), kThreads, 0, s, H, sxy, ncy, g->rowStart);

        // scratch: scan tile counter + look-back state (+ error flag, + residual words)
        const int64_t scanTiles = (g->ncells + kScanBlock * kScanItems - 1) / (kScanBlock * kScanItems);
        const int64_t nState = std::max<int64_t>(scanTiles, 1);
        // + counter, err[4], frameOff[F + 1]: err and the frame offsets are read back together
        unsigned long long* state = dalloc<unsigned long long>(A, nState + 3 + (F + 2) / 2, s);
        unsigned* counter = reinterpret_cast<unsigned*>(state + nState);
        int* err = reinterpret_cast<int*>(state + nState + 1);
        g->frameOff = reinterpret_cast<int*>(state + nState + 3);
        zero_words(state, (nState + 3) * sizeof(unsigned long long), s);
        g->vid = dalloc<int>(A, N, s);
        uint64_t* keysCap = dalloc<uint64_t>(A, N, s);
        int* mCap = dalloc<int>(A, N + kVecPad, s);
        g->cellOff = dalloc<int>(A, g->ncells + 1, s);
        CellGeom geo{F, H, W, ncx, ncy, g->colStart, g->rowStart};
        uint8_t* lutL = dalloc<uint8_t>(A, 65536, s);
        uint8_t* lutUV = dalloc<uint8_t>(A, 65536, s);
        LAUNCH(k_bin_lut, 256, 256, 0, s, 256.0 * sl, lutL);
        // D = 3: the chroma bins are held at 0 (reading #27)
        LAUNCH(k_bin_lut, 256, 256, 0, s, g->dims == 3 ? 1e300 : 256.0 * suv, lutUV);
        g->perm = dalloc<uint8_t>(A, (size_t)g->ncells * kCellMaxPx, s);
        int* cellCnt = dalloc<int>(A, g->ncells, s);
        unsigned long long* heads = dalloc<unsigned long long>(A, g->ncells, s);
        g->heads = heads;  // kept: the splat ranks its sorted pixels from it
        const int cellBlocks = grid_for(g->ncells * 32, 256, 1 << 20);
        LAUNCH(k_grid_sort, cellBlocks, 256, 0, s, rgb, geo, lutL, lutUV, g->ncells, cellCnt, heads, g->perm, err);
        LAUNCH(k_scan_excl, (unsigned)std::max<int64_t>(scanTiles, 1), kScanBlock, 0, s, cellCnt, g->ncells, g->cellOff,
               counter, state, (int64_t)ncx * ncy, g->frameOff);
        LAUNCH(k_grid_write, cellBlocks, 256, 0, s, rgb, geo, lutL, lutUV, g->ncells, g->cellOff, heads, g->perm,
               keysCap, mCap, g->vid);

        // No host synchronisation anywhere in the build: every vertex array is sized by a rigorous
        // capacity known on the host (level 0: M ≤ N; level k: M_k ≤ min(M_{k−1}, cells_k × codes_k)),
        // every kernel reads the data-dependent counts (frame and level offsets) from device memory,
        // and launch sizes derive from the capacities (grid-stride loops).  The exact counts are read
        // back only by the synchronous query / export calls (ensure_sizes).
        g->err = err;
        g->keys = keysCap;
        g->m = mCap;
        const int64_t M = N;  // level-0 capacity (and the channel stride of every vertex vector)
        g->M = M;
        g->maxFrameM = std::max<int64_t>(1, (int64_t)H * W / 3);  // launch-size heuristic only

        // The pyramid and the tree order need only the keys and the frame and cell offsets, not n:
        // they run on a side stream `sp` concurrently with Alg. 1, whose launches are latency-bound
        // (configs[2]: 1.35 → 1.30 ms per build + solve).  Until the PDL trigger change (kernels
        // no longer trigger their dependents at entry, fbs_common.cuh) the concurrent pyramid
        // slowed the bench batch's Alg. 1 more than it hid (5.06 vs 4.99 ms per step); since, it
        // pays there too: 4.925 → 4.825 ms.
        // FBS_PYR_FORK (A/B): 0 serial, 1 fork after the neighbour search, 2 before it.
        static const int pyrForkEnv = [] {
            const char* e = std::getenv("FBS_PYR_FORK");
            return (e && e[0]) ? std::atoi(e) : -1;
        }();
        const int pyrFork = pyrForkEnv >= 0 ? pyrForkEnv : 1;
        const bool pyrSide = pyrFork != 0 && want_pyr && cap.size() > 1;
        cudaStream_t sp = s;
        cudaEvent_t pyrFork0 = nullptr, pyrJoin = nullptr;
        auto fork_pyramid = [&]() {
            sp = group_stream(dev, s, 2);
            pyrForked = true;
            ck(cudaEventCreateWithFlags(&pyrFork0, cudaEventDisableTiming), "event");
            ck(event_record(pyrFork0, s), "event");
            ck(stream_wait(sp, pyrFork0), "wait");
            cudaEventDestroy(pyrFork0);
        };
        if (pyrSide && pyrFork == 2) fork_pyramid();

        g->nbr = dalloc<int4>(A, M + kVecPad, s);
        // Phase boundaries of the build are fully serialised launches: one unbroken programmatic
        // (PDL) chain through the whole build faulted on B200 (a pyramid or tree kernel read data of
        // the level-0 build that was not yet visible), while serialising any of these boundaries
        // fixed it (tests/test_gpu_ops.py ragged shapes; scripts/pdl_bisect.sh)
        pdl_break(s, 32);
        LAUNCH(k_grid_neighbours, grid_for(g->ncells * 32, 256, 1 << 20), 256, 0, s, g->keys, g->cellOff, ncx, ncy,
               g->ncells, g->nbr, err);
        if (pyrSide && pyrFork == 1) fork_pyramid();

        // ---- Alg. 1 (reading #5: fixed n_bistoch iterations)
        g->n = dalloc<float>(A, M + kVecPad, s);
        float* ntmp = dalloc<float>(A, M + kVecPad, s);
        float* cur = ntmp;
        float* nxt = g->n;
        if (g->n_bistoch % 2 == 0) std::swap(cur, nxt);  // make the last write land in g->n
        int bsPerSM = 4;  // 4 × (512 threads, 2 × 25 KB stages) per SM: 5.57 → 5.43 ms per bench step against 3
        if (const char* e = std::getenv("FBS_BS_BLOCKS")) bsPerSM = std::max(1, std::min(4, std::atoi(e)));  // A/B
        // frames in Gb groups on Gb streams (frames are independent: no neighbour crosses a frame), so
        // one group's kernel boundaries overlap the other's work; each group's launches take 1/Gb of
        // the resident blocks
        // round 1 (host-sized launches): 1: 5.46, 2: 5.38, 4: 5.34, 8: 5.41 ms per bench step;
        // round 2 (device-read frame ranges, arena layout): 1: 5.29, 2: 5.23, 4: 5.33 ms
        int Gb = std::min(F, 2);
        if (const char* e = std::getenv("FBS_BS_GROUPS")) Gb = std::max(1, std::min(F, std::atoi(e)));  // A/B
        // dynamic chunk scheduling (k_bistoch): one counter per launch, zeroed before the fork.
        // Off since the PDL trigger change and the pyramid beside Alg. 1: static chunks measured
        // 4.813 -> 4.798 ms per bench step, configs[2] 1.113 -> 1.096 ms (FBS_BS_DYNAMIC=1: A/B)
        static const bool bsDynamic = [] {
            const char* e = std::getenv("FBS_BS_DYNAMIC");  // A/B
            return e && e[0] == '1';
        }();
        unsigned* bsCtr = nullptr;
        if (bsDynamic && g->n_bistoch > 0) {
            bsCtr = dalloc<unsigned>(A, (size_t)g->n_bistoch * Gb, s);
            zero_words(bsCtr, (size_t)g->n_bistoch * Gb * sizeof(unsigned), s);
        }
        cudaEvent_t bsFork = nullptr;
        std::vector<cudaEvent_t> bsJoin(Gb, nullptr);
        if (Gb > 1) {
            ck(cudaEventCreateWithFlags(&bsFork, cudaEventDisableTiming), "event");
            ck(event_record(bsFork, s), "event");
        }
        const int sms = g_num_sms > 0 ? g_num_sms : 148;
        for (int gi = 0; gi < Gb; ++gi) {
            const int f0 = (int)((int64_t)F * gi / Gb), f1 = (int)((int64_t)F * (gi + 1) / Gb);
            cudaStream_t sg = s;
            if (Gb > 1) {
                sg = group_stream(dev, s, gi);
                ck(stream_wait(sg, bsFork), "wait");
            }
            float* c2 = cur;
            float* n2 = nxt;
            // the group's vertex range [frameOff[f0], frameOff[f1]) is read on the device; the grid
            // is sized by its pixel count (an upper bound of its vertices)
            const int64_t chunksCap = ((int64_t)(f1 - f0) * H * W + kBsChunk - 1) / kBsChunk + 1;
            const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(chunksCap, std::max(1, bsPerSM * sms / Gb)));
            for (int it = 0; it < g->n_bistoch && f1 > f0; ++it) {
                LAUNCH(k_bistoch, blocks, kBsThreads, kBsSmem, sg, g->nbr, g->m, c2, n2, g->frameOff, F, f0, f1, it == 0,
                       (float)(2 * g->dims), bsCtr ? bsCtr + (size_t)it * Gb + gi : nullptr);
                std::swap(c2, n2);
            }
            if (Gb > 1) {
                ck(cudaEventCreateWithFlags(&bsJoin[gi], cudaEventDisableTiming), "event");
                ck(event_record(bsJoin[gi], sg), "event");
            }
        }
        if (Gb > 1) {
            for (int gi = 0; gi < Gb; ++gi) {
                ck(stream_wait(s, bsJoin[gi]), "wait");
                cudaEventDestroy(bsJoin[gi]);
            }
            cudaEventDestroy(bsFork);
        }
        if (g->n_bistoch == 0) {  // n = 1 (Alg. 1 with no iterations)
            const float one = 1.f;
            int bits;
            std::memcpy(&bits, &one, 4);
            LAUNCH(k_fill_words, grid_for(M), kThreads, 0, s, reinterpret_cast<int*>(g->n), (int64_t)M, bits);
        }

        // ---- pyramid (Supp. Sec. 2), levels 1 .. Lmax-1 (capacities: level_caps)
        const int Lmax = (int)cap.size();
        g->capH = cap;
        const uint64_t* keysK = g->keys;
        const int* cellOffK = g->cellOff;
        int ncxK = ncx, ncyK = ncy;
        // frame offsets of every level in one [Lmax][F + 1] array (row 0: level 0), used by the
        // hierarchy kernels as is
        int* lvAll = dalloc<int>(A, (size_t)Lmax * (F + 1), sp);
        copy_words(g->frameOff, lvAll, (F + 1) * sizeof(int), sp);
        unsigned long long* pyrScratch = (Lmax > 1) ? dalloc<unsigned long long>(A, 2 * (size_t)M + 2, sp) : nullptr;
        int* pyrRank = (Lmax > 1) ? dalloc<int>(A, M, sp) : nullptr;  // parent rank of each sorted child
        // scan look-back states and (tile counter, scratch bump) pairs of every level: one zeroing
        std::vector<int64_t> st2Off(Lmax + 1, 0);
        for (int k = 1; k < Lmax; ++k) {
            const int64_t nc = (int64_t)F * (((ncx - 1) >> k) + 1) * (((ncy - 1) >> k) + 1);
            st2Off[k + 1] = st2Off[k] + std::max<int64_t>(1, (nc + kScanBlock * kScanItems - 1) / (kScanBlock * kScanItems)) + 1;
        }
        unsigned long long* st2All = nullptr;
        if (Lmax > 1) {
            st2All = dalloc<unsigned long long>(A, st2Off[Lmax], sp);
            zero_words(st2All, st2Off[Lmax] * sizeof(unsigned long long), sp);
        }
        for (int k = 1; k < Lmax; ++k) {
            Level& L = g->lv[k];
            L.ncx = ((ncx - 1) >> k) + 1;
            L.ncy = ((ncy - 1) >> k) + 1;
            L.ncells = (int64_t)F * L.ncx * L.ncy;
            L.M = cap[k];
            L.keys = dalloc<uint64_t>(A, cap[k], sp);
            L.cellOff = dalloc<int>(A, L.ncells + 1, sp);
            L.parent = dalloc<int>(A, cap[k - 1], sp);
            L.childStart = dalloc<int>(A, cap[k] + 1, sp);
            L.childList = dalloc<int>(A, cap[k - 1], sp);
            L.count = dalloc<int>(A, cap[k], sp);
            if (k >= 2) L.cnt1 = dalloc<int>(A, cap[k], sp);
            int* cnt2 = dalloc<int>(A, L.ncells, sp);
            const int64_t st2n = std::max<int64_t>(1, (L.ncells + kScanBlock * kScanItems - 1) / (kScanBlock * kScanItems));
            unsigned long long* st2 = st2All + st2Off[k];
            unsigned* ctr2 = reinterpret_cast<unsigned*>(st2 + st2n);  // scan tile counter, scratch bump
            if (k == 1 || pdl_every_level()) pdl_break(sp, 32);
            LAUNCH(k_pyr_sort, grid_for(L.ncells * 32, 256, 1 << 20), 256, 0, sp, keysK, cellOffK, ncxK, ncyK, L.ncx,
                   L.ncy, L.ncells, ctr2 + 1, pyrScratch, L.childList, pyrRank, cnt2);
            LAUNCH(k_scan_excl, (unsigned)st2n, kScanBlock, 0, sp, cnt2, L.ncells, L.cellOff, ctr2, st2,
                   (int64_t)L.ncx * L.ncy, lvAll + (size_t)k * (F + 1));
            LAUNCH(k_pyr_write, grid_for(L.ncells * 32, 256, 1 << 20), 256, 0, sp, keysK, cellOffK, ncxK, ncyK, L.ncx,
                   L.ncy, L.ncells, L.cellOff, L.childList, pyrRank, L.keys, L.parent, L.childStart,
                   k >= 2 ? g->lv[k - 1].count : nullptr, L.count, k >= 3 ? g->lv[k - 1].cnt1 : nullptr,
                   k >= 2 ? L.cnt1 : nullptr);
            keysK = L.keys;
            cellOffK = L.cellOff;
            ncxK = L.ncx;
            ncyK = L.ncy;
        }
        g->bistoch_residual = -1.f;  // computed on request (fbs_grid_export)
        g->L = Lmax;  // levels carried by the hierarchy kernels; each frame's own count is on the device
        g->has_pyramid = want_pyr;
        g->lvFrameOffDev = lvAll;  // rows 0 .. L − 1 (row 0 = level 0)
        // per-frame level counts (first level with a single vertex, reading #8) and, with a pyramid,
        // the prefix-scan tiles of the tree-ordered level 1 — both computed on the device
        const int L = Lmax;
        g->frameLevels = dalloc<int>(A, F, sp);
        pdl_break(sp, 32);
        LAUNCH(k_frame_levels, (F + 255) / 256, 256, 0, sp, lvAll, F, L, g->frameLevels);
        // ---- tree order of the pyramid (tree_kernels.cuh): depth-first positions of the level-0 and
        // level-1 vertices, so every coarse subtree is one contiguous level-1 range
        if (L > 1) {
            TreeOrder& T = g->tree;
            const int64_t M1 = cap[1];
            const int top = L - 1;
            std::vector<int*> cnt1(L, nullptr);  // level-1 descendants of levels ≥ 2
            for (int k = 2; k < L; ++k) cnt1[k] = g->lv[k].cnt1;
            std::vector<int2*> start(L, nullptr);
            for (int k = 1; k < L; ++k) start[k] = dalloc<int2>(A, cap[k], sp);
            for (int k = 2; k < L; ++k) T.rng[k] = dalloc<int2>(A, cap[k], sp);
            T.tord0 = dalloc<int>(A, M, sp);
            T.csT = dalloc<int>(A, M1 + 1, sp);
            T.tord1 = dalloc<int>(A, M1, sp);
            T.parent0T = dalloc<int>(A, M, sp);
            LAUNCH(k_tree_top, 1, 256, 0, sp, g->lvFrameOffDev, F, top, start[top], top >= 2 ? T.rng[top] : nullptr,
                   top >= 2 ? cnt1[top] : nullptr);
            for (int k = top; k >= 1; --k) {
                const int km1 = k - 1;
                LAUNCH(k_tree_down, grid_for(cap[k]), kThreads, 0, sp, km1, g->lv[k].childStart, g->lv[k].childList,
                       lvAll + (size_t)k * (F + 1) + F, start[k], km1 >= 1 ? g->lv[km1].count : nullptr,
                       km1 >= 2 ? cnt1[km1] : nullptr, km1 >= 1 ? start[km1] : nullptr,
                       km1 >= 2 ? T.rng[km1] : nullptr, T.tord0, T.tord1, T.csT);
            }
            LAUNCH(k_tree_finish, grid_for(M), kThreads, 0, sp, g->lv[1].parent, start[1], lvAll + F, lvAll + (F + 1) + F,
                   T.parent0T, T.csT);
            if (top >= 3) {  // ancestor tables of the level-2 vertices
                const int64_t M2 = cap[2];
                T.ancId = dalloc<int>(A, (size_t)(top - 2) * M2, sp);
                T.ancRng = dalloc<int2>(A, (size_t)(top - 2) * M2, sp);
                HierArgs hb{};
                hb.L = L;
                hb.M2 = M2;
                for (int k = 2; k < L; ++k) {
                    hb.lv[k].M = cap[k];
                    hb.lv[k].parent = (k + 1 < L) ? g->lv[k + 1].parent : nullptr;
                    hb.lv[k].rng = T.rng[k];
                }
                LAUNCH(k_tree_anc, grid_for(M2), kThreads, 0, sp, hb, lvAll + 2 * (size_t)(F + 1) + F, T.ancId, T.ancRng);
            }
            // prefix-scan tiles: kScanTile level-1 positions, never crossing a frame (device-built)
            T.nTiles1 = (int)((M1 + kScanTile - 1) / kScanTile + F);  // capacity
            T.tileFrameOff = dalloc<int>(A, F + 1, sp);
            T.tileRange = dalloc<int2>(A, T.nTiles1, sp);
            T.tileFrame = dalloc<int>(A, T.nTiles1, sp);
            LAUNCH(k_scan_tiles, F, 256, 0, sp, lvAll + (F + 1), F, T.tileFrameOff, T.tileRange, T.tileFrame);
        }
        // launch-size heuristics for the level-1 / level-2 kernels: each level typically holds ~1/5
        // of the vertices below it (Appendix A of SURVEY.md; 1/4 here to err towards more blocks)
        g->maxFrameM1 = std::max<int64_t>(1, std::min<int64_t>(g->maxFrameM / 4, L > 1 ? cap[1] : 1));
        g->maxFrameM2 = std::max<int64_t>(1, std::min<int64_t>(g->maxFrameM1 / 4, L > 2 ? cap[2] : 1));
        if (sp != s) {  // join the pyramid's side stream
            ck(cudaEventCreateWithFlags(&pyrJoin, cudaEventDisableTiming), "event");
            ck(event_record(pyrJoin, sp), "event");
            ck(stream_wait(s, pyrJoin), "wait");
            cudaEventDestroy(pyrJoin);
        }
    } catch (...) {
        if (pyrForked) cudaStreamSynchronize(group_stream(dev, s, 2));  // error path: drain it first
        free_all(g->allocs, s);
        for (auto& b : g->uploads) pinned_put(b, s);
        delete g;
        throw;
    }
    *out = g;
}

// The exact sizes of a grid (vertex and level counts per frame, levels per frame) live on the
// device; the synchronous query and export calls read them back once (one synchronisation of the
// grid's stream) and check the build's internal invariants.
static void ensure_sizes(fbs_grid g) {
    if (g->sized) return;
    cudaStream_t s = g->stream;
    const int F = g->F, L = g->L;
    std::vector<int> lv((size_t)L * (F + 1)), fl(F);
    int errh[4];
    ck(memcpy_async(lv.data(), g->lvFrameOffDev, lv.size() * sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
    ck(memcpy_async(fl.data(), g->frameLevels, F * sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
    ck(memcpy_async(errh, g->err, sizeof(errh), cudaMemcpyDeviceToHost, s), "d2h");
    ck(cudaStreamSynchronize(s), "sync");
    if (errh[0] & 1) throw Err(FBS_ELIMIT, "a sigma_xy cell holds more than 64 pixels");
    if (errh[0] & 6) throw Err(FBS_ECUDA, "internal grid-build check failed (code " + std::to_string(errh[0]) + ")");
    g->frameOffH.assign(lv.begin(), lv.begin() + F + 1);
    g->Mx = lv[F];
    g->levelMx.assign(L, 0);
    g->Lx = 1;
    for (int f = 0; f < F; ++f) g->Lx = std::max(g->Lx, fl[f]);
    for (int k = 0; k < L; ++k) g->levelMx[k] = lv[(size_t)k * (F + 1) + F];
    g->frameLevelsH = fl;
    g->sized = true;
}

// ===================================================================================== solve
namespace {

VecArgs make_args(fbs_system S, PcgScalars sc, float* x, const float* b) {
    fbs_grid g = S->g;
    VecArgs a{};
    a.K = S->K;
    a.BPF = S->BPF;
    a.nf = g->F;
    a.M = g->M;
    a.lam = (float)S->lam;
    a.frameOff = g->frameOff;
    a.nbr = g->nbr;
    a.n = g->n;
    a.sc = S->sc;
    a.diagA = S->diagA;
    a.x = x;
    a.r = S->rh;
    a.dn = S->dn;
    a.ldn = (g->M + 3) & ~3ll;
    a.q = S->qh;
    a.s = S->sh;
    a.b = b;
    a.mu0 = S->mu0;
    a.partial = S->partial;
    a.counters = S->counters;
    a.ksplit = 0;
    a.sc_ = sc;
    a.tol_mode = S->o.mode == FBS_MODE_TOL;
    a.tol2 = S->o.tol * S->o.tol;
    a.max_iters = (S->o.mode == FBS_MODE_TOL) ? S->o.max_iters : S->o.iters;
    return a;
}

// ---- hierarchical machinery (tree_kernels.cuh)
HierArgs make_hier(fbs_system S, int C, double alpha, double beta) {
    fbs_grid g = S->g;
    HierArgs h{};
    h.L = g->L;
    h.F = g->F;
    h.C = C;
    h.nt = g->tree.nTiles1;  // capacity (the lift reads the group's tile range on the device)
    h.nfG = g->F;
    h.f0 = 0;
    // FBS_COARSE_TILES (tests): frames with more level-1 scan tiles take the lift's tile-base path
    h.coarseTiles = kCoarseTiles;
    if (const char* e = std::getenv("FBS_COARSE_TILES")) h.coarseTiles = std::max(0, std::min(kCoarseTiles, std::atoi(e)));
    for (int k = 0; k < g->L; ++k) {
        HLevel& v = h.lv[k];
        v.M = (k == 0) ? g->M : g->lv[k].M;
        if (k > 0) {
            const Level& L = g->lv[k];
            v.childStart = L.childStart;
            v.childList = L.childList;
            v.count = L.count;
            v.mu = (k >= 2) ? S->mu[k] : nullptr;
            v.rng = g->tree.rng[k];
        }
        v.parent = (k + 1 < g->L) ? g->lv[k + 1].parent : nullptr;
    }
    h.frameLevels = g->frameLevels;
    h.lvFrameOff = g->lvFrameOffDev;
    h.alpha = alpha;
    h.beta = beta;
    for (int k = 0; k < kMaxLevels; ++k) h.zw[k] = std::pow(alpha, -(beta + (double)k));
    const TreeOrder& T = g->tree;
    h.tord0 = T.tord0;
    h.ancRng = T.ancRng;
    h.ancMult = S->ancMult;
    h.M2 = (g->L > 2) ? g->lv[2].M : 0;
    h.csT = T.csT;
    h.parent0T = T.parent0T;
    h.tileFrameOff = T.tileFrameOff;
    h.tileFrame = T.tileFrame;
    h.tileRange = T.tileRange;
    h.nTiles1 = T.nTiles1;
    h.M0 = g->M;
    h.M1 = g->lv[1].M;
    h.mu1T = S->mu[1];
    h.buf1T = S->buf1T;
    h.locT = S->locT;
    h.tileAgg = S->tileAgg;
    h.tileBase = S->tileBase;
    h.tcount = S->tcount;
    h.acc1T = S->acc1T;
    h.partial2 = S->partial2;
    h.counters = S->counters2;
    h.bpf2 = S->bpf2;
    return h;
}

const char* mode_name(int m) {
    static const char* n[] = {"PCG", "PDA", "INIT", "PLAIN"};
    return n[m];
}

// The channel-split view of `a` (block_unit): K > 1 right-hand sides get BPFs blocks each.
VecArgs split_args(fbs_system S, const VecArgs& a) {
    VecArgs as = a;
    if (a.K > 1) {
        as.ksplit = 1;
        as.BPF = S->BPFs;
    }
    return as;
}
int vec_blocks(const VecArgs& a) { return a.nf * a.BPF * (a.ksplit ? a.K : 1); }

// P of the level-0 input in0 [C][M0] to tree-ordered level 1 + prefix scan (k_tree_lift).
// PCG and hierarchical init with K > 1 channels: channel-split kernels (one channel per block group).
// active: PCG mode, the per-(frame, channel) flags of the running solve (inactive channels skip)
template <int MODE>
void tree_lift(fbs_system S, const HierArgs& h, const float* in0, cudaStream_t s, const int* active = nullptr) {
    static const std::string name = std::string("k_tree_lift<") + mode_name(MODE) + ">";
    // work items walked grid-stride (the group's tile count, ≤ capacity h.nt, is on the device);
    // the grid is the resident capacity of the kernel, shared by the concurrent frame groups
    const bool ks = (MODE == HIER_PCG && h.C > 1) || (MODE == HIER_INIT && h.C > 2);
    auto kern = ks ? k_tree_lift<MODE, true> : k_tree_lift<MODE, false>;
    static int occ[2] = {0, 0};
    if (!occ[ks]) {
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[ks], kern, kScanTile, 0), "occupancy");
        occ[ks] = std::max(1, occ[ks]);
    }
    // (more blocks than resident slots measured faster than a resident-sized grid: 38.7 µs at 8 per
    // SM vs 54 µs at the occupancy limit split between the frame groups)
    int perSM = 8;
    if (const char* e = std::getenv("FBS_LIFT_GRID")) perSM = std::max(1, std::atoi(e));  // A/B
    const int64_t cap = std::max<int64_t>(1, (int64_t)g_num_sms * perSM);
    const int64_t items = (int64_t)h.nt * (ks ? h.C : 1);
    LAUNCH_AS(name.c_str(), kern, (int)std::max<int64_t>(1, std::min<int64_t>(items, cap)), kScanTile, 0, s, h, in0,
              active);
}

// coarse values and their projection onto level 2 (k_tree_coarse)
template <int MODE>
void tree_coarse(fbs_system S, const HierArgs& h, const VecArgs& a, int first, cudaStream_t s) {
    static const std::string name = std::string("k_tree_coarse<") + mode_name(MODE) + ">";
    const bool ks = (MODE == HIER_PCG && h.C > 1) || (MODE == HIER_INIT && h.C > 2);
    auto kern = ks ? k_tree_coarse<MODE, true> : k_tree_coarse<MODE, false>;
    // ks: the finish reads the split level-0 kernel's partials (BPFs per (frame, channel))
    if (MODE == HIER_PCG && S->bpf2g > 0) {  // small problems: G = 8 lanes per level-2 vertex
        HierArgs hg = h;
        hg.bpf2 = S->bpf2g;
        auto kg = ks ? k_tree_coarse<HIER_PCG, true, 8> : k_tree_coarse<HIER_PCG, false, 8>;
        LAUNCH_AS(name.c_str(), kg, a.nf * hg.bpf2 * (ks ? h.C : 1), 256, 0, s, hg, ks ? split_args(S, a) : a, first);
        return;
    }
    LAUNCH_AS(name.c_str(), kern, a.nf * S->bpf2 * (ks ? h.C : 1), 256, 0, s, h, ks ? split_args(S, a) : a, first);
}

// level-0 output (k_tree_level0)
template <int MODE>
void tree_level0(fbs_system S, const HierArgs& h, const VecArgs& a, const float* in0, float* out0, int first,
                 cudaStream_t s) {
    static const std::string name = std::string("k_tree_level0<") + mode_name(MODE) + ">";
    if ((MODE == HIER_PCG || MODE == HIER_INIT) && a.K > 1) {
        const VecArgs as = split_args(S, a);
        auto kern = k_tree_level0<MODE, true>;
        LAUNCH_AS(name.c_str(), kern, vec_blocks(as), kThreads, 0, s, h, as, in0, out0, first);
    } else {
        auto kern = k_tree_level0<MODE, false>;
        VecArgs a2 = a;  // the PCG direction kernel has no reduction: its own blocks per frame
        if (MODE == HIER_PCG) a2.BPF = S->BPFl0;
        LAUNCH_AS(name.c_str(), kern, a2.nf * a2.BPF, kThreads, 0, s, h, a2, in0, out0, first);
    }
}

// where k_hier_level0 stores w = mask∘r: nowhere when r is already masked (S->rMasked; the lift
// then reads r itself)
bool w_is_r(fbs_system S) {
    static const bool off = std::getenv("FBS_WRITE_W") != nullptr;  // A/B: always materialise w
    return S->rMasked && !off;
}
float* lift_w0(fbs_system S) { return w_is_r(S) ? nullptr : S->w0; }

// level-0 PCG input w = mask∘r (+ ρ_0, ‖r‖² partials) (k_hier_level0)
template <int SRC, bool LAST>
void hier_level0(fbs_system S, const VecArgs& a, cudaStream_t s) {
    static const char* src_names[] = {"UPDATE", "RESID", "RESID0"};
    static const std::string name =
        std::string("k_hier_level0<") + src_names[SRC] + (LAST ? ",LAST>" : ">");
    if (a.K > 1) {
        const VecArgs as = split_args(S, a);
        auto kern = k_hier_level0<SRC, LAST, true>;
        LAUNCH_AS(name.c_str(), kern, vec_blocks(as), kThreads, 0, s, as, lift_w0(S));
    } else {
        auto kern = k_hier_level0<SRC, LAST, false>;
        LAUNCH_AS(name.c_str(), kern, a.nf * S->BPF, kThreads, 0, s, a, lift_w0(S));
    }
}

// s = M⁻¹_hier r and d = s + βd after the level-0 kernel (Alg. 2 lines 10-14)
void hier_precond_direction(fbs_system S, const VecArgs& a, const HierArgs& h, int first, cudaStream_t s) {
    tree_lift<HIER_PCG>(S, h, w_is_r(S) ? a.r : S->w0, s, a.sc_.active);
    tree_coarse<HIER_PCG>(S, h, a, first, s);
    tree_level0<HIER_PCG>(S, h, a, nullptr, nullptr, first, s);
}

// The launch arguments of frames [f0, f0 + nf): per-frame and per-tile pointers shifted so that
// the kernels (which index frames from blockIdx) see the group as frames 0 … nf − 1.
void restrict_frames(fbs_system S, int f0, int nf, VecArgs& a, HierArgs& h) {
    fbs_grid g = S->g;
    const int K = S->K;
    a.nf = nf;
    a.frameOff += f0;
    a.counters += (size_t)f0 * K;
    a.partial += (size_t)f0 * std::max(S->BPF, S->BPFk) * 2 * K;
    PcgScalars& q = a.sc_;
    q.rho += f0 * K;
    q.alpha += f0 * K;
    q.xalpha += f0 * K;
    q.beta += f0 * K;
    q.bb += f0 * K;
    q.rr += f0 * K;
    q.active += f0 * K;
    q.iters += f0 * K;
    q.status += f0 * K;
    // the group's tiles: [tileFrameOff[f0], tileFrameOff[f0 + nf]) on the device; a capacity for
    // the launch size from its frames' share
    h.nt = (int)std::min<int64_t>(g->tree.nTiles1, (int64_t)g->tree.nTiles1 * nf / std::max(1, g->F) + nf + 1);
    h.nfG = nf;
    h.f0 = f0;
    h.lvFrameOff += f0;  // [L][F+1] row-major: k·(F+1) + f0 + f
    h.frameLevels += f0;
    h.tileFrameOff += f0;  // tile ids stay global (tileFrameOff[f] − tileFrameOff[0] is group-local)
    h.partial2 += (size_t)f0 * std::max(S->bpf2, S->bpf2g) * h.C;
    h.counters += f0;
}


// a9: x = Sᵀy; 4 pixels per thread when the frame size and x allow it
void slice(fbs_grid g, const float* y, int64_t M, int K, int planar, float* x, cudaStream_t s) {
    const int64_t HW = (int64_t)g->H * g->W;
    if (HW % 4 == 0 && ((uintptr_t)x & 15) == 0 && ((uintptr_t)g->vid & 15) == 0 && g->F <= 65535) {
        const dim3 grid((unsigned)((HW / 4 + kThreads - 1) / kThreads), (unsigned)g->F);
        LAUNCH(k_slice4, grid, kThreads, 0, s, g->vid, y, M, K, HW, planar, x);
    } else {
        LAUNCH(k_slice, grid_for(g->N), kThreads, 0, s, g->vid, y, M, K, g->F, HW, planar, x);
    }
}

// q = A d and α: k_spmv2 (K = 1), k_spmv_kjoint / k_spmv2_split (K > 1)
// K > 1: the channel-split kernel (default) or, with FBS_SPMV_K=joint, the channel-joint one
// (one nbr read per vertex for all channels; 89 vs 19 µs per launch on configs[3])
bool spmv_kjoint() {
    const char* e = std::getenv("FBS_SPMV_K");
    return e && std::strcmp(e, "joint") == 0;
}
VecArgs with_bpf(VecArgs a, int bpf) {
    a.BPF = bpf;
    return a;
}
void spmv(fbs_system S, const VecArgs& a, cudaStream_t s) {
    if (a.K > 1 && spmv_kjoint()) {
        LAUNCH(k_spmv_kjoint, a.nf * S->BPFk, kThreads, 0, s, a.BPF == S->BPFk ? a : with_bpf(a, S->BPFk));
        return;
    }
    const VecArgs as = split_args(S, a);
    auto kern = as.ksplit ? k_spmv2_split : k_spmv2;
    LAUNCH_AS("k_spmv2", kern, vec_blocks(as), kThreads, 0, s, as);
}

// One PCG iteration (Alg. 2 lines 6-14): SpMV + α; update (+ M⁻¹ and ρ, β); direction.
// Hierarchical: ρ = rᵀM⁻¹r comes from the lift, and Pᵀ is fused with d = s + βd
// (tree_kernels.cuh).  last: the final FIXED-mode iteration needs no new direction.
void pcg_iteration(fbs_system S, const VecArgs& a, const HierArgs& h, int it, bool last, cudaStream_t s) {
    const VecArgs as = split_args(S, a);
    const int nb = vec_blocks(as);
    if (S->useHierP) {
        spmv(S, a, s);
        if (last) {
            hier_level0<HSRC_UPDATE, true>(S, a, s);
        } else {
            hier_level0<HSRC_UPDATE, false>(S, a, s);
            hier_precond_direction(S, a, h, 0, s);
        }
    } else {
        LAUNCH(k_direction2, nb, kThreads, 0, s, as, it == 0);
        spmv(S, a, s);
        LAUNCH(k_update, nb, kThreads, 0, s, as);
    }
}

// Alg. 2 lines 1-4 for the frames of `a`.
void pcg_start(fbs_system S, const VecArgs& a, const HierArgs& h, bool x_zero, cudaStream_t s) {
    const VecArgs as = split_args(S, a);
    const int nb = vec_blocks(as);
    const int FKg = a.nf * S->K;  // a group's scalars start at its first frame (restrict_frames)
    LAUNCH(k_init_scalars, (FKg + 255) / 256, 256, 0, s, a.sc_, FKg, 1);  // each view has its own count
    if (S->useHierP) {
        // Alg. 2 lines 2-4: r = b − A x, ρ = rᵀM⁻¹r (lift), d = s = M⁻¹r (project)
        if (x_zero) hier_level0<HSRC_RESID0, false>(S, a, s);
        else hier_level0<HSRC_RESID, false>(S, a, s);
        hier_precond_direction(S, a, h, 1, s);
    } else {
        auto k1 = k_residual0<true>;
        auto k2 = k_residual0<false>;
        if (x_zero) LAUNCH(k1, nb, kThreads, 0, s, as);
        else LAUNCH(k2, nb, kThreads, 0, s, as);
        // d = s (Alg. 2 line 3) is the first iteration's k_direction2
    }
}

// TOL iterations 1 … as a device-side loop: a graph whose conditional while node runs one PCG
// iteration plus k_tol_cond per trip, launched once on s (no host polls, no overshoot, no host
// synchronisation).  Returns false (nothing launched) if the graph cannot be built.
bool tol_graph(fbs_system S, const VecArgs& a, cudaStream_t s) {
    // off by default: measured on configs[0,1,3] it is no faster than the host-polled loop (graph
    // instantiation per solve costs what the polls cost; the device-side loop adds ~2 µs per trip)
    const char* e = std::getenv("FBS_TOL_GRAPH");
    if (!e || e[0] != '1') return false;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaStream_t cs = group_stream(dev, s, 7);  // capture stream (nothing executes on it)
    bool ok = false;
    if (cudaGraphCreate(&graph, 0) == cudaSuccess) {
        cudaGraphConditionalHandle h;
        cudaGraphNodeParams p = {};
        cudaGraphNode_t node;
        int* it = dalloc<int>(S->allocs, 1, s);
        zero_words(it, sizeof(int), s);
        if (cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault) == cudaSuccess) {
            p.type = cudaGraphNodeTypeConditional;
            p.conditional.handle = h;
            p.conditional.type = cudaGraphCondTypeWhile;
            p.conditional.size = 1;
            if (cudaGraphAddNode(&node, graph, nullptr, 0, &p) == cudaSuccess &&
                cudaStreamBeginCaptureToGraph(cs, p.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                              cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
                bool cap = true;
                try {
                    pcg_iteration(S, a, S->hP, 1, false, cs);
                    LAUNCH(k_tol_cond, 1, 32, 0, cs, h, a.sc_.n_active, it, S->o.max_iters + 1);
                } catch (...) {
                    cap = false;
                }
                cudaGraph_t body = nullptr;
                if (cudaStreamEndCapture(cs, &body) != cudaSuccess) cap = false;
                ok = cap && cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess &&
                     cudaGraphLaunch(exec, s) == cudaSuccess;
            }
        }
    }
    cudaGetLastError();  // a failed attempt leaves no sticky error: fall back to host polling
    if (exec) cudaGraphExecDestroy(exec);  // freed when the launch completes
    if (graph) cudaGraphDestroy(graph);
    return ok;
}

// TOL iterations 1 … inside a CUDA graph the CALLER is capturing on s: a conditional while node
// is added at the capture's current position (its body: one PCG iteration + k_tol_cond, captured
// on a side stream), and the capture continues after it.  A TOL solve is then replayable like a
// FIXED one, with per-channel stopping on the device and no host polls.  Returns false if s is
// not capturing.
bool tol_loop_in_capture(fbs_system S, const VecArgs& a, const HierArgs& h, cudaStream_t s, int side) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    ck(cudaStreamIsCapturing(s, &st), "cudaStreamIsCapturing");
    if (st != cudaStreamCaptureStatusActive) return false;
    int dev = 0;
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    int* it = dalloc<int>(S->allocs, 1, s);
    zero_words(it, sizeof(int), s);  // captured: re-zeroed at every replay
    cudaGraph_t graph = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    ck(cudaStreamGetCaptureInfo(s, &st, nullptr, &graph, &deps, &ndeps), "cudaStreamGetCaptureInfo");
    cudaGraphConditionalHandle hc;
    ck(cudaGraphConditionalHandleCreate(&hc, graph, 1, cudaGraphCondAssignDefault), "conditional handle");
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = hc;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    ck(cudaGraphAddNode(&node, graph, deps, ndeps, &p), "conditional node");
    ck(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies), "capture deps");
    cudaStream_t cs = group_stream(dev, s, 8 + side);  // body capture stream (nothing executes on it)
    ck(cudaStreamBeginCaptureToGraph(cs, p.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                     cudaStreamCaptureModeRelaxed),
       "body capture");
    try {
        pdl_break(cs, 8);
        pcg_iteration(S, a, h, 1, false, cs);
        LAUNCH(k_tol_cond, 1, 32, 0, cs, hc, a.sc_.n_active, it, S->o.max_iters + 1);
    } catch (...) {
        cudaGraph_t body = nullptr;
        cudaStreamEndCapture(cs, &body);
        throw;
    }
    cudaGraph_t body = nullptr;
    ck(cudaStreamEndCapture(cs, &body), "body capture end");
    pdl_break(s, 4);
    return true;
}

// TOL polling for one or more independent PCGs (frame groups) on their own streams: each gets
// chunks of 4 iterations in turn, and the host reads each one's active count (a copy kernel
// into mapped pinned memory) one chunk behind; a group whose count reached 0 gets no more.
struct PcgRun {
    VecArgs a;
    HierArgs h;
    cudaStream_t s;
};
// The host's view of a TOL run after a chunk: the active count and, for a single (frame,
// channel), ‖b‖² and the last ‖r‖² (k_tol_probe copies them into mapped pinned memory).
struct TolProbe {
    int n_active;
    int pad;
    double bb, rr;
};
// Host-polled TOL loop: each run enqueues a chunk of iterations and a probe, then reads the probe
// of the chunk before (one chunk behind, so the GPU never waits for the host).  A run of a single
// (frame, channel) sizes its next chunk from the residual's observed rate of decrease: near
// convergence the chunks shrink to the predicted remainder (≥ 1), so fewer iterations are
// launched past the stopping point (they change nothing — the retired channel's kernels skip — but
// each costs its launches).  The iterates and the stopping iteration are the same for any chunking.
void tol_poll(fbs_system S, std::vector<PcgRun>& runs) {
    const int n = (int)runs.size();
    static const int chunk = [] {
        const char* e = std::getenv("FBS_TOL_CHUNK");  // A/B
        // 6 with the adaptive shrink near convergence (configs[0] 0.864 -> 0.828 ms against 4)
        return (e && e[0]) ? std::max(1, std::min(64, std::atoi(e))) : 6;
    }();
    static const bool adapt = [] {
        const char* e = std::getenv("FBS_TOL_ADAPT");  // A/B: 0 = fixed chunks
        return !(e && e[0] == '0');
    }();
    PinnedBlock pb = pinned_get(2 * n * sizeof(TolProbe));
    TolProbe* pin = static_cast<TolProbe*>(pb.p);
    std::vector<cudaEvent_t> ev(2 * n, nullptr);
    std::vector<int> done(n, 1), slot(n, 0), pending(n, -1), at(2 * n, 0);
    std::vector<char> fin(n, 0);
    // the last two (iteration, ‖r‖²) observations of single-(frame, channel) runs
    std::vector<int> it1(n, -1), it2(n, -1);
    std::vector<double> rr1(n, 0.0), rr2(n, 0.0), bbv(n, 0.0);
    try {
        for (auto& e : ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        for (int left = n; left > 0;) {
            for (int r = 0; r < n; ++r) {
                if (fin[r]) continue;
                const VecArgs& a = runs[r].a;
                const bool single = a.nf * a.K == 1;
                int nit = std::min(chunk, S->o.max_iters - done[r]);
                if (adapt && single && it1[r] >= 0 && it2[r] > it1[r] && rr2[r] > 0.0 && rr2[r] < rr1[r]) {
                    // geometric model of ‖r‖² from the last two observations
                    const double q = std::pow(rr2[r] / rr1[r], 1.0 / (it2[r] - it1[r]));
                    const double target = a.tol2 * bbv[r];
                    if (q < 1.0 && target > 0.0) {
                        const double m = std::ceil(std::log(target / rr2[r]) / std::log(q));
                        const double rem = m - (double)(done[r] - it2[r]);
                        if (rem < nit) nit = std::max(1, (int)std::max(1.0, rem));
                    }
                }
                for (int i = 0; i < nit; ++i) pcg_iteration(S, runs[r].a, runs[r].h, done[r] + i, false, runs[r].s);
                done[r] += nit;
                at[2 * r + slot[r]] = done[r];
                LAUNCH(k_tol_probe, 1, 32, 0, runs[r].s, a.sc_.n_active, single ? a.sc_.bb : nullptr,
                       single ? a.sc_.rr : nullptr, reinterpret_cast<int*>(&pin[2 * r + slot[r]]));
                ck(event_record(ev[2 * r + slot[r]], runs[r].s), "event");
            }
            for (int r = 0; r < n; ++r) {
                if (fin[r]) continue;
                bool stop = done[r] >= S->o.max_iters;
                if (pending[r] >= 0) {
                    const int ps = 2 * r + pending[r];
                    ck(cudaEventSynchronize(ev[ps]), "event sync");
                    if (pin[ps].n_active == 0) stop = true;
                    it1[r] = it2[r];
                    rr1[r] = rr2[r];
                    it2[r] = at[ps];
                    rr2[r] = pin[ps].rr;
                    bbv[r] = pin[ps].bb;
                }
                pending[r] = slot[r];
                slot[r] ^= 1;
                if (stop) {
                    fin[r] = 1;
                    --left;
                }
            }
        }
        for (auto& r : runs) ck(cudaStreamSynchronize(r.s), "sync");
    } catch (...) {
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        pinned_put(pb, runs[0].s);
        throw;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    pinned_put(pb, runs[0].s);
}

// Full PCG (Alg. 2) from the state in a.x (right-hand side a.b); x_zero: x0 = 0.
// With several frames, the frames are split into groups whose PCGs run on their own streams
// (forked from and joined back to `s`): the frames are independent systems, so one group's
// latency-bound kernels overlap the other's bandwidth-bound ones.  TOL mode: each group has its
// own active count and stops on its own (tol_poll).
void run_pcg(fbs_system S, const VecArgs& a, bool x_zero, cudaStream_t s) {
    fbs_grid g = S->g;
    // Jacobi on small frames: the whole PCG of each (frame, channel) in one CTA (k_pcg_small);
    // FBS_SMALL_PX sets the per-frame pixel bound (0 = off); FBS_SPMV_K=joint (the A/B switch of
    // the channel-joint SpMV) keeps the multi-kernel path
    static const int64_t small_px = [] {
        const char* e = std::getenv("FBS_SMALL_PX");
        return (e && e[0]) ? (int64_t)std::atoll(e) : (int64_t)kSmallPx;
    }();
    // larger frames up to FBS_CLUSTER_PX pixels: a cluster of kPcgCluster CTAs per (frame, channel)
    static const int64_t cluster_px = [] {
        const char* e = std::getenv("FBS_CLUSTER_PX");
        return (e && e[0]) ? (int64_t)std::atoll(e) : (int64_t)kClusterPx;
    }();
    // (measured, scripts/ab_cluster_sizes.py: the cluster path wins up to 240x320 at any K, ties
    // the multi-kernel path at 375x500 with K = 21 and loses 2x there with K ≤ 3, whose 8-24
    // CTAs leave most SMs idle; so beyond kClusterPxAnyK pixels it needs ≥ 16 (frame, channel)s)
    const int64_t HWf = (int64_t)g->H * g->W;
    const int FK = a.nf * S->K;
    const bool cluster_ok = HWf <= cluster_px && (HWf <= kClusterPxAnyK || FK >= 16);
    if (!S->useHierP && (HWf <= small_px || cluster_ok) && !spmv_kjoint()) {
        LAUNCH(k_init_scalars, (FK + 255) / 256, 256, 0, s, a.sc_, FK, 1);
        if (HWf <= small_px) LAUNCH(k_pcg_small, FK, kSmallThreads, 0, s, a, (int)x_zero);
        else LAUNCH(k_pcg_cluster, FK * kPcgCluster, kSmallThreads, 0, s, a, (int)x_zero);
        return;
    }
    const int G = std::min(S->nGroups, g->F);
    const bool tol = S->o.mode == FBS_MODE_TOL;
    if (G > 1) {
        int dev = 0;
        ck(cudaGetDevice(&dev), "cudaGetDevice");
        cudaEvent_t fork;
        std::vector<cudaEvent_t> join(G);
        ck(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming), "event");
        ck(event_record(fork, s), "event");
        std::vector<PcgRun> runs;
        for (int gi = 0; gi < G; ++gi) {
            const int f0 = (int)((int64_t)g->F * gi / G), f1 = (int)((int64_t)g->F * (gi + 1) / G);
            cudaStream_t sg = group_stream(dev, s, gi);
            ck(stream_wait(sg, fork), "wait");
            VecArgs ag = a;
            HierArgs hg = S->hP;
            restrict_frames(S, f0, f1 - f0, ag, hg);
            ag.sc_.n_active = a.sc_.n_active + 1 + gi;  // the group's own active count
            pcg_start(S, ag, hg, x_zero, sg);
            if (tol) {
                pcg_iteration(S, ag, hg, 0, false, sg);
                runs.push_back({ag, hg, sg});
            } else {
                for (int i = 0; i < S->o.iters; ++i) pcg_iteration(S, ag, hg, i, i == S->o.iters - 1, sg);
            }
        }
        if (tol && S->o.max_iters > 1) {
            // inside the caller's graph capture: a device-side loop per group, else host polls
            bool captured = true;
            for (size_t r = 0; r < runs.size() && captured; ++r)
                captured = tol_loop_in_capture(S, runs[r].a, runs[r].h, runs[r].s, (int)r);
            if (!captured) tol_poll(S, runs);
        }
        for (int gi = 0; gi < G; ++gi) {
            cudaStream_t sg = group_stream(dev, s, gi);
            ck(cudaEventCreateWithFlags(&join[gi], cudaEventDisableTiming), "event");
            ck(event_record(join[gi], sg), "event");
            ck(stream_wait(s, join[gi]), "wait");
            cudaEventDestroy(join[gi]);
        }
        cudaEventDestroy(fork);
        return;
    }
    pcg_start(S, a, S->hP, x_zero, s);
    if (!tol) {
        for (int i = 0; i < S->o.iters; ++i) pcg_iteration(S, a, S->hP, i, i == S->o.iters - 1, s);
        return;
    }
    // TOL: device-side per-channel stopping; the host polls the active count one chunk behind
    // (FBS_TOL_GRAPH=1: the loop runs on the device instead, as a CUDA graph with a conditional
    // while node).
    pcg_iteration(S, a, S->hP, 0, false, s);  // iteration 0 (Jacobi: d = s) outside the loop
    if (S->o.max_iters <= 1 || tol_loop_in_capture(S, a, S->hP, s, 0) || tol_graph(S, a, s)) return;
    std::vector<PcgRun> runs{{a, S->hP, s}};
    tol_poll(S, runs);
}

// the per-(frame, channel) PCG scalars of FK pairs: 6 double and 3 int arrays of FK, + the active
// count and one count per frame group (≤ 8), in scalars_doubles(FK) doubles at d (zeroed by the caller)
size_t scalars_doubles(int FK) { return (size_t)6 * FK + ((size_t)3 * FK + 1 + 8 + 1) / 2 + 1; }
PcgScalars scalars_at(double* d, int FK) {
    PcgScalars p;
    p.rho = d;
    p.alpha = d + FK;
    p.xalpha = d + 2 * (size_t)FK;
    p.beta = d + 3 * (size_t)FK;
    p.bb = d + 4 * (size_t)FK;
    p.rr = d + 5 * (size_t)FK;
    int* i = reinterpret_cast<int*>(d + 6 * (size_t)FK);
    p.active = i;
    p.iters = i + FK;
    p.status = i + 2 * (size_t)FK;
    p.n_active = i + 3 * (size_t)FK;
    return p;
}

PcgScalars alloc_scalars(AllocList& A, int FK, cudaStream_t s) {
    // one allocation, zeroed by one launch
    const size_t nD = scalars_doubles(FK);
    double* d = dalloc<double>(A, nD, s);
    PcgScalars p;
    p.rho = d;
    p.alpha = d + FK;
    p.xalpha = d + 2 * (size_t)FK;
    p.beta = d + 3 * (size_t)FK;
    p.bb = d + 4 * (size_t)FK;
    p.rr = d + 5 * (size_t)FK;
    int* i = reinterpret_cast<int*>(d + 6 * (size_t)FK);
    p.active = i;
    p.iters = i + FK;
    p.status = i + 2 * (size_t)FK;
    p.n_active = i + 3 * (size_t)FK;
    zero_words(d, nD * sizeof(double), s);
    return p;
}

void validate_opts(const fbs_solve_opts& o, fbs_grid g) {
    if (o.precond != FBS_PRECOND_JACOBI && o.precond != FBS_PRECOND_HIER) throw Err(FBS_EINVAL, "bad precond");
    if (o.init != FBS_INIT_FLAT && o.init != FBS_INIT_HIER && o.init != FBS_INIT_ZERO) throw Err(FBS_EINVAL, "bad init");
    if (o.mode != FBS_MODE_FIXED && o.mode != FBS_MODE_TOL) throw Err(FBS_EINVAL, "bad mode");
    if (o.mode == FBS_MODE_FIXED && o.iters < 0) throw Err(FBS_EINVAL, "iters must be >= 0");
    if (o.mode == FBS_MODE_TOL && (o.max_iters < 0 || !(o.tol >= 0.0))) throw Err(FBS_EINVAL, "bad tol/max_iters");
    if ((o.precond == FBS_PRECOND_HIER || o.init == FBS_INIT_HIER) && !g->has_pyramid)
        throw Err(FBS_EINVAL, "hierarchical precond/init need a grid built with build_pyramid = 1");
    if (o.precond == FBS_PRECOND_HIER && !(o.precond_alpha > 0.0)) throw Err(FBS_EINVAL, "precond_alpha must be > 0");
    if (o.init == FBS_INIT_HIER && !(o.init_alpha > 0.0)) throw Err(FBS_EINVAL, "init_alpha must be > 0");
    if (!(o.lowrank_eps >= 0.0 && o.lowrank_eps < 1.0)) throw Err(FBS_EINVAL, "lowrank_eps must be in [0, 1)");
}

}  // namespace

static void solve_impl(fbs_grid g, const float* t, int K, const float* c, double lam, const fbs_solve_opts* opts,
                       float* x, float* y, fbs_system* sys_out, cudaStream_t s) {
    if (!g || !t || !c || !x) throw Err(FBS_EINVAL, "null pointer");
    if (K < 1 || K > kMaxK) throw Err(FBS_EINVAL, "K must be in [1, 64]");
    if (!(lam > 0.0) || !std::isfinite(lam)) throw Err(FBS_EINVAL, "lambda must be finite and > 0");
    fbs_solve_opts o;
    if (opts) o = *opts; else fbs_default_solve_opts(&o);
    validate_opts(o, g);
    int dev = 0;
    device_setup(&dev);
    pdl_break(s);

    const bool lowrank = o.lowrank_eps > 0.0 && K > 1;
    if (lowrank && sys_out) throw Err(FBS_EINVAL, "a low-rank solve keeps no system (sys_out must be NULL)");

    fbs_system S = new fbs_system_s();
    try {
        S->g = g;
        S->lam = lam;
        S->o = o;
        S->stream = s;
        const int64_t M = g->M;
        const int F = g->F;
        auto& A = S->allocs;
        {  // one up-front allocation for the system's buffers (see arena_reserve)
            const size_t M4 = (size_t)M * 4, C = (size_t)K + 1;
            size_t b = M4 * (C + 2 + 8 * (size_t)K + C + 2 * (size_t)K) + (size_t)16 * kVecPad * 16 + (1 << 20);
            if (g->L > 1) {
                const size_t c1 = g->capH.size() > 1 ? (size_t)g->capH[1] : 0;
                b += 16 * (C + 1) * c1 + 16 * (C + 1) * ((size_t)g->tree.nTiles1 + 1);  // + the side PDA's level-1 scratch
                for (size_t k = 1; k < g->capH.size(); ++k) b += 4 * (size_t)g->capH[k] + 256;
                if (g->capH.size() > 3) b += 4 * (g->capH.size() - 3) * (size_t)g->capH[2];
            }
            arena_reserve(A, b, s);
        }
        // launch geometry of the per-frame kernels: BPF blocks per frame
        // 16 blocks of 256 threads per SM: two full SMs' worth, so that each of the two frame
        // groups of a FIXED-mode solve (run_pcg) fills the GPU on its own and the groups overlap
        // in the dependent-launch gaps (8: 6.60 ms, 16: 6.21 ms per bench step; one group: equal)
        int occ = 16;
        if (const char* e = std::getenv("FBS_BPF_OCC")) occ = std::max(1, std::min(64, std::atoi(e)));  // A/B
        // at least vpt vertices per thread: single-frame solves get fewer, fuller blocks (round 1,
        // configs[1,2]: 3.09 → 2.79 and 1.54 → 1.46 ms at 2); the bench batch is capped by
        // occupancy.  Re-measured after the PDL trigger change: 3 for K = 1 (configs[1] 2.13 →
        // 2.03, configs[2] 1.14 → 1.12 ms; 4 slows configs[0]), 6 for K > 1, where the channel-split
        // kernels carry the PCG and the unsplit ones want fewer blocks (configs[3] 1.87 → 1.72 ms)
        int vpt = K > 1 ? 6 : 3;
        if (const char* e = std::getenv("FBS_VPT")) vpt = std::max(1, std::min(64, std::atoi(e)));  // A/B
        const int64_t want = (g->maxFrameM + (int64_t)kThreads * vpt - 1) / ((int64_t)kThreads * vpt);
        const int64_t cap = std::max<int64_t>(1, ((int64_t)g_num_sms * std::max(occ, 1) + F - 1) / F);
        S->BPF = (int)std::max<int64_t>(1, std::min(want, cap));
        {  // k_tree_level0<PCG>: 24 resident blocks' worth per SM (5.28 -> 5.25 ms per bench step)
            int occ0 = 24;
            if (const char* e = std::getenv("FBS_L0_OCC")) occ0 = std::max(1, std::min(64, std::atoi(e)));  // A/B
            S->BPFl0 = (int)std::max<int64_t>(1, std::min(want, ((int64_t)g_num_sms * occ0 + F - 1) / F));
        }
        {
            const char* e = std::getenv("FBS_PCG_GROUPS");  // A/B measurement: 1 disables the split
            S->nGroups = (e && e[0]) ? std::max(1, std::min(8, std::atoi(e))) : 2;
        }
        // b and Sc in one allocation, [b_0 .. b_{K−1}, Sc] with channel stride M: the hierarchical
        // init lifts exactly these K + 1 channels, so it reads them in place
        float* bIn = dalloc<float>(A, (size_t)(K + 1) * M + kVecPad, s);
        S->sc = bIn + (size_t)K * M;
        CellGeom geo{F, g->H, g->W, g->ncx, g->ncy, g->colStart, g->rowStart};
        // every buffer that must start at zero, in one block zeroed by one launch: the input-check
        // flags (FBS_ST_NEG_CONF / FBS_ST_NONFINITE from the splats), the last-block counters, the
        // lift's per-(frame, channel) tile counters, the forward PCG scalars, the low-rank Gram counters
        const size_t zInts = 8 + (size_t)2 * F * K + (size_t)(K + 1) * F + F + F;
        const size_t zDoubles = scalars_doubles(F * K);
        double* zblk = dalloc<double>(A, zDoubles + (zInts + 1) / 2, s);
        zero_words(zblk, (zDoubles + (zInts + 1) / 2) * sizeof(double), s);
        S->fwd = scalars_at(zblk, F * K);
        int* zi = reinterpret_cast<int*>(zblk + zDoubles);
        S->inflags = zi;
        S->counters = reinterpret_cast<unsigned*>(zi + 8);  // [F][K] VecArgs, [K][F] HierArgs
        S->counters2 = S->counters + (size_t)F * K;
        S->tcount = S->counters + (size_t)2 * F * K;        // [K + 1][F] (k_tree_lift)
        unsigned* zctr = S->tcount + (size_t)(K + 1) * F;    // [F] (k_gram)
        unsigned* pdaTcount = zctr + F;                      // [F] (the side PDA lift)
        // a4: splat Sc, b = S(c∘t)
        LAUNCH(k_splat<true>, grid_for(g->ncells * 32, 256, 1 << 20), 256, 0, s, geo, g->cellOff, g->heads, g->perm, c, t,
               K, M, S->sc, bIn, S->inflags);
        // optional low-rank reduction of B (Supp. §4): Kc reduced channels
        int Kc = K;
        double* lrRt = nullptr;
        if (lowrank) {
            const int P = K * (K + 1) / 2;
            const int bpfG = std::min(S->BPF, 64);
            double* part = dalloc<double>(A, (size_t)F * bpfG * P, s);
            unsigned* ctr = zctr;
            double* G = dalloc<double>(A, (size_t)F * K * K, s);
            double* T = dalloc<double>(A, (size_t)F * K * K, s);
            lrRt = dalloc<double>(A, (size_t)F * K * K, s);
            int* tF = dalloc<int>(A, F, s);
            LAUNCH(k_gram, F * bpfG, 256, 0, s, bIn, M, K, g->frameOff, bpfG, part, ctr, G);
            LAUNCH(k_pchol, F, 64, 0, s, G, K, o.lowrank_eps, tF, lrRt, T);
            // no host synchronisation: the reduced solve carries K channels; those at or above a
            // frame's kept rank t_f get zero right-hand sides (zero columns of T), so they are
            // converged at iteration 0 and every PCG kernel skips them (per-(frame, channel) flags)
            S->lr_rank = tF;
            S->b = dalloc<float>(A, (size_t)Kc * M, s);
            LAUNCH(k_reduce_rhs, F * S->BPF, kThreads, 0, s, bIn, M, K, Kc, g->frameOff, S->BPF, T, S->b);
        } else {
            S->b = bIn;
        }
        S->K = Kc;
        S->C = Kc + 1;
        const size_t KM = (size_t)Kc * M;
        S->diagA = dalloc<float>(A, M, s);
        S->mu0 = dalloc<float>(A, M, s);
        S->xh = dalloc<float>(A, KM, s);
        S->rh = dalloc<float>(A, KM, s);
        S->dn = dalloc<float2>(A, (size_t)Kc * ((M + 3) & ~3ll) + kVecPad, s);
        S->qh = dalloc<float>(A, KM, s);
        S->sh = dalloc<float>(A, KM, s);
        const bool hierP = o.precond == FBS_PRECOND_HIER && g->L > 1;  // L = 1: hier ≡ Jacobi / flat
        const bool hierI = o.init == FBS_INIT_HIER && g->L > 1;
        S->useHierP = hierP;
        S->rMasked = true;  // b = S(c∘t) and the initial residual are 0 on dead vertices (reading #6)
        if (hierP || hierI) {
            const int C = S->C;
            const int64_t M1 = g->lv[1].M;
            const int nT = g->tree.nTiles1;
            S->w0 = dalloc<float>(A, (size_t)C * M, s);
            S->buf1T = dalloc<float>(A, (size_t)C * M1, s);
            S->acc1T = dalloc<float>(A, (size_t)C * M1, s);
            S->locT = dalloc<double>(A, (size_t)C * M1, s);
            S->tileAgg = dalloc<double>(A, (size_t)C * nT, s);
            S->tileBase = dalloc<double>(A, (size_t)C * nT, s);
            const int64_t want2 = ((g->L > 2 ? g->maxFrameM2 : g->maxFrameM1) + 255) / 256;
            int occ2 = 8;
            if (const char* e = std::getenv("FBS_BPF2_OCC")) occ2 = std::max(1, std::min(64, std::atoi(e)));  // A/B
            const int64_t cap2 = std::max<int64_t>(1, ((int64_t)g_num_sms * occ2 + F - 1) / F);
            S->bpf2 = (int)std::max<int64_t>(1, std::min(want2, cap2));
            // the PCG coarse pass with 8 lanes per level-2 vertex when all of them fit in about
            // two resident waves (single frames: configs[1, 2]); FBS_COARSE_G=1 / 8 forces (A/B)
            {
                const char* e = std::getenv("FBS_COARSE_G");
                const int64_t lanes = (int64_t)F * (g->L > 2 ? g->maxFrameM2 : 0) * 8;
                // (K = 1 only: with the channel split the blocks × channels outgrow the work — configs[3]
                // hierarchical 1.98 → 2.27 ms)
                const bool small = g->L > 2 && Kc == 1 && lanes <= 2ll * g_num_sms * 4 * 256;
                const bool on = e ? std::atoi(e) == 8 && g->L > 2 : small;
                const int64_t capg = std::max<int64_t>(1, ((int64_t)g_num_sms * 4 + F - 1) / F);
                S->bpf2g = on ? (int)std::max<int64_t>(1, std::min<int64_t>((lanes / F + 255) / 256, capg)) : 0;
            }
            S->partial2 = dalloc<double>(A, (size_t)F * std::max(S->bpf2, S->bpf2g) * C, s);
            if (hierP) {
                for (int k = 1; k < g->L; ++k) S->mu[k] = dalloc<float>(A, g->lv[k].M, s);
            }
            if (g->L > 3) S->ancMult = dalloc<float>(A, (size_t)(g->L - 3) * g->lv[2].M, s);
        }
        {  // channel-split kernels: at least vptS vertices per thread (more blocks in flight per SM)
            int vptS = 4;
            if (const char* e = std::getenv("FBS_VPT_SPLIT")) vptS = std::max(1, std::min(64, std::atoi(e)));  // A/B
            const int64_t wantS = (g->maxFrameM + (int64_t)kThreads * vptS - 1) / ((int64_t)kThreads * vptS);
            S->BPFs = (int)std::max<int64_t>(
                1, std::min<int64_t>({S->BPF, wantS, ((int64_t)g_num_sms * occ + (int64_t)F * Kc - 1) / ((int64_t)F * Kc)}));
        }
        // channel-joint SpMV (K > 1): a warp per vertex, ≥ 4 vertices per warp, within the
        // partials' [F][BPF] capacity
        S->BPFk = (int)std::max<int64_t>(
            1, std::min<int64_t>(((int64_t)g_num_sms * occ + F - 1) / F, (g->maxFrameM + 31) / 32));
        S->partial = dalloc<double>(A, (size_t)F * std::max(S->BPF, S->BPFk) * 2 * Kc, s);
        if (hierP || hierI) S->hP = make_hier(S, Kc, o.precond_alpha, o.precond_beta);

        // a5: assemble (+ flat/zero init)
        VecArgs a = make_args(S, S->fwd, S->xh, S->b);
        const int init_mode = (o.init == FBS_INIT_HIER && !hierI) ? FBS_INIT_FLAT : o.init;
        const VecArgs as = split_args(S, a);
        LAUNCH(k_assemble, vec_blocks(as), kThreads, 0, s, as, S->diagA, S->mu0, init_mode, S->fwd);
        // a6/a7: hierarchical preconditioner multipliers μ_k = z_w P(1) / P(diag A), and init
        // (running the two concurrently on two streams measured slower: 5.10 vs 4.99 ms per step)
        // With both, the multipliers run on a side stream beside the init (their own level-1
        // scratch; the two share only the grid's read-only tree): since the PDL trigger change
        // (fbs_common.cuh) this overlap pays — FBS_PDA_SIDE=0 serialises (A/B).
        static const bool pdaSideEnv = [] {
            const char* e = std::getenv("FBS_PDA_SIDE");
            return !(e && e[0] == '0');
        }();
        const bool pdaSide = pdaSideEnv && hierP && hierI;
        cudaStream_t spda = s;
        if (hierP) {
            HierArgs h = make_hier(S, 1, o.precond_alpha, o.precond_beta);
            if (pdaSide) {
                const int64_t M1 = g->lv[1].M;
                const int nT = g->tree.nTiles1;
                h.buf1T = dalloc<float>(A, (size_t)M1, s);
                h.locT = dalloc<double>(A, (size_t)M1, s);
                h.tileAgg = dalloc<double>(A, (size_t)nT, s);
                h.tileBase = dalloc<double>(A, (size_t)nT, s);
                h.tcount = pdaTcount;
                spda = group_stream(dev, s, 3);
                cudaEvent_t ev;
                ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
                ck(event_record(ev, s), "event");
                ck(stream_wait(spda, ev), "wait");
                cudaEventDestroy(ev);
            }
            tree_lift<HIER_PDA>(S, h, S->diagA, spda);  // (P diag A)_1 (diag A is the lift's input)
            tree_coarse<HIER_PDA>(S, h, a, 0, spda);
        }
        if (hierI) {
            HierArgs h = make_hier(S, Kc + 1, o.init_alpha, o.init_beta);
            const float* w0i = bIn;  // [b, Sc] in place (above); the low-rank b is its own array
            if (lowrank) {
                LAUNCH(k_fill_init_w0, grid_for(M), kThreads, 0, s, S->b, S->sc, M, Kc, S->w0);
                w0i = S->w0;
            }
            if (g->L > 3) {
                auto km = k_tree_anc_mult<HIER_INIT>;
                LAUNCH_AS("k_tree_anc_mult<INIT>", km, F * S->bpf2, kThreads, 0, s, h, g->tree.ancId, S->ancMult);
            }
            tree_lift<HIER_INIT>(S, h, w0i, s);
            tree_coarse<HIER_INIT>(S, h, a, 0, s);
            tree_level0<HIER_INIT>(S, h, a, w0i, S->xh, 0, s);
        }
        if (pdaSide) {  // join: the PCG's multipliers come from the side stream
            cudaEvent_t ev;
            ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
            ck(event_record(ev, spda), "event");
            ck(stream_wait(s, ev), "wait");
            cudaEventDestroy(ev);
        }
        if (hierP && g->L > 3) {
            auto km = k_tree_anc_mult<HIER_PCG>;
            LAUNCH_AS("k_tree_anc_mult<PCG>", km, F * S->bpf2, kThreads, 0, s, S->hP, g->tree.ancId, S->ancMult);
        }
        if (sys_out) {  // the initial guess is kept for fbs_system_export only
            S->y0 = dalloc<float>(A, KM, s);
            ck(memcpy_async(S->y0, S->xh, KM * sizeof(float), cudaMemcpyDeviceToDevice, s), "d2d");
        }
        // a8: PCG
        run_pcg(S, a, false, s);
        // low rank: Y = Ỹ R̃ (Supp. §4)
        const float* ysol = S->xh;
        if (lowrank) {
            float* yfull = dalloc<float>(A, (size_t)K * M, s);
            LAUNCH(k_expand, F * S->BPF, kThreads, 0, s, S->xh, M, K, Kc, g->frameOff, S->BPF, lrRt, yfull);
            ysol = yfull;
        }
        // a9: slice
        slice(g, ysol, M, K, 1, x, s);
        if (y) LAUNCH(k_export_vk, grid_for((size_t)K * M), kThreads, 0, s, ysol, g->frameOff + F, (int64_t)0, M, K, y);
    } catch (...) {
        free_all(S->allocs, s);
        delete S;
        throw;
    }
    if (sys_out) {
        *sys_out = S;
    } else {
        free_all(S->allocs, s);
        delete S;
    }
}

// Alg. 3: IRLS around the solver with Geman–McClure weights.
static void robust_impl(fbs_grid g, const float* t, int K, const float* c_init, double lam, const fbs_solve_opts* opts,
                        double sigma_gm, int n_irls, float* x, float* c_out, cudaStream_t s) {
    if (!g || !t || !c_init || !x) throw Err(FBS_EINVAL, "null pointer");
    if (K != 1) throw Err(FBS_EINVAL, "the robust solver takes scalar targets (K = 1)");
    if (!(sigma_gm > 0.0) || !std::isfinite(sigma_gm)) throw Err(FBS_EINVAL, "sigma_gm must be finite and > 0");
    if (n_irls < 1) throw Err(FBS_EINVAL, "n_irls must be >= 1");
    AllocList tmp;
    float* c = (n_irls > 1 || c_out) ? (c_out ? c_out : dalloc<float>(tmp, g->N, s)) : nullptr;
    try {
        const float* cur = c_init;
        const float s2 = (float)(sigma_gm * sigma_gm);
        for (int i = 0; i < n_irls; ++i) {
            solve_impl(g, t, 1, cur, lam, opts, x, nullptr, nullptr, s);  // line 3
            if (i + 1 < n_irls || c_out) {                                // lines 4-5
                LAUNCH(k_gm_weight, grid_for(g->N), kThreads, 0, s, x, t, g->N, s2, c);
                cur = c;
            }
        }
    } catch (...) {
        free_all(tmp, s);
        throw;
    }
    free_all(tmp, s);
}

// Domain-transform post-filter (reading #28): N iterations of a row pass and a column pass.
static void dt_impl(const uint8_t* rgb, int F, int H, int W, const float* in, int K, double sigma_s, double sigma_r,
                    int n_iters, float* out, cudaStream_t s) {
    if (!rgb || !in || !out) throw Err(FBS_EINVAL, "null pointer");
    if (F < 1 || H < 1 || W < 1 || K < 1 || K > kMaxK) throw Err(FBS_EINVAL, "bad sizes");
    if (H > 16384 || W > 16384) throw Err(FBS_EINVAL, "lines longer than 16384 pixels are not supported");
    if (!(sigma_s > 0.0) || !(sigma_r > 0.0) || n_iters < 1) throw Err(FBS_EINVAL, "sigma_s, sigma_r > 0, n_iters >= 1");
    int dev = 0;
    device_setup(&dev);
    pdl_break(s);
    AllocList tmp;
    try {
        const size_t NP = (size_t)F * H * W, NS = NP * K;
        float* Dx = dalloc<float>(tmp, NP, s);
        float* Dy = dalloc<float>(tmp, NP, s);
        if ((W & 3) == 0 && ((uintptr_t)rgb & 3) == 0)  // four pixels per thread, word loads
            LAUNCH(k_dt_dist4, dim3((W / 4 + kThreads - 1) / kThreads, std::min(F * H, 65535)), kThreads, 0, s, rgb, F, H,
                   W, (float)(sigma_s / sigma_r), Dx, Dy);
        else
            LAUNCH(k_dt_dist, dim3((W + kThreads - 1) / kThreads, std::min(F * H, 65535)), kThreads, 0, s, rgb, F, H, W,
                   (float)(sigma_s / sigma_r), Dx, Dy);
        if (out != in) ck(memcpy_async(out, in, NS * sizeof(float), cudaMemcpyDeviceToDevice, s), "d2d");
        const size_t perWarp = 2 * (size_t)(W + 32) * sizeof(float);
        const int nw = (int)std::max<size_t>(1, std::min<size_t>(8, (64 * 1024) / perWarp));
        const size_t smem = perWarp * nw;
        if (smem > 48 * 1024)
            ck(cudaFuncSetAttribute((const void*)k_dt_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
               "smem attr");
        const int64_t lines = (int64_t)F * K * H;
        // rows of ≥ 256 pixels (W % 4 = 0): two warps per row (k_dt_rows2; FBS_DT_ROWS1=1 for A/B)
        const bool rows2 = (W % 4 == 0) && W >= 256 && !std::getenv("FBS_DT_ROWS1");
        const size_t smem2 = 8 * 2 * (size_t)(((W + 1) / 2 + 3) / 4 * 4 + 33) * sizeof(float);
        const int rowBlocks2 = (int)std::max<int64_t>(1, std::min<int64_t>((lines + 3) / 4, 148 * 32));
        if (rows2 && smem2 > 48 * 1024)
            ck(cudaFuncSetAttribute((const void*)k_dt_rows2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2),
               "smem attr");
        const int rowBlocks = (int)std::max<int64_t>(1, std::min<int64_t>((lines + nw - 1) / nw, 148 * 32));
        // column passes: register-resident columns (H ≤ 1536), else row passes on the transpose
        // (FBS_DT_COLS=t / 1 for A/B: the transpose path / the in-place column kernel)
        const char* dtc = std::getenv("FBS_DT_COLS");
        const bool colsReg = H <= kDtColChunks * kDtColRows && !(dtc && dtc[0]);
        const bool viaT = !colsReg && !(dtc && dtc[0] == '1');
        float* sT = nullptr;
        float* DyT = nullptr;
        const size_t perWarpT = 2 * (size_t)(H + 32) * sizeof(float);
        const int nwT = (int)std::max<size_t>(1, std::min<size_t>(8, (64 * 1024) / perWarpT));
        const size_t smemT = perWarpT * nwT;
        const int64_t linesT = (int64_t)F * K * W;
        const int rowBlocksT = (int)std::max<int64_t>(1, std::min<int64_t>((linesT + nwT - 1) / nwT, 148 * 32));
        const dim3 tb(32, 8), tgN((W + 31) / 32, (H + 31) / 32, F * K), tgT((H + 31) / 32, (W + 31) / 32, F * K);
        if (viaT) {
            sT = dalloc<float>(tmp, NS, s);
            DyT = dalloc<float>(tmp, NP, s);
            LAUNCH(k_dt_transpose, dim3((W + 31) / 32, (H + 31) / 32, F), tb, 0, s, Dy, DyT, H, W);
            if (std::max(smem, smemT) > 48 * 1024)
                ck(cudaFuncSetAttribute((const void*)k_dt_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)std::max(smem, smemT)),
                   "smem attr");
        }
        const int colThreads = 32 * std::max(1, std::min(32, H));  // ≥ 1 row per warp chunk
        const int64_t colTiles = (int64_t)F * K * ((W + 31) / 32);
        const int colBlocks = (int)std::max<int64_t>(1, std::min<int64_t>(colTiles, 148 * 8));
        for (int i = 1; i <= n_iters; ++i) {
            const double sig = sigma_s * std::sqrt(3.0) * std::pow(2.0, n_iters - i) / std::sqrt(std::pow(4.0, n_iters) - 1.0);
            const float lna = (float)(-std::sqrt(2.0) / sig);  // ln a_i
            if (rows2) LAUNCH(k_dt_rows2, rowBlocks2, 256, smem2, s, out, Dx, F, K, H, W, lna);
            else LAUNCH(k_dt_rows, rowBlocks, 32 * nw, smem, s, out, Dx, F, K, H, W, lna);
            if (colsReg) {
                static const int colsPer = [] {  // A/B: FBS_DT_COLSPER = 4, 8 or 16
                    const char* e = std::getenv("FBS_DT_COLSPER");
                    const int v = e ? std::atoi(e) : 8;
                    return (v == 4 || v == 16) ? v : 8;
                }();
                const int64_t tiles = (int64_t)F * K * ((W + colsPer - 1) / colsPer);
                const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, 148 * 32));
                if (colsPer == 16) LAUNCH_AS("k_dt_cols_reg", k_dt_cols_reg<16>, blocks, 1024, 0, s, out, Dy, F, K, H, W, lna);
                else if (colsPer == 4) LAUNCH_AS("k_dt_cols_reg", k_dt_cols_reg<4>, blocks, 256, 0, s, out, Dy, F, K, H, W, lna);
                else LAUNCH_AS("k_dt_cols_reg", k_dt_cols_reg<8>, blocks, 512, 0, s, out, Dy, F, K, H, W, lna);
            } else if (viaT) {
                LAUNCH(k_dt_transpose, tgN, tb, 0, s, out, sT, H, W);
                LAUNCH(k_dt_rows, rowBlocksT, 32 * nwT, smemT, s, sT, DyT, F, K, W, H, lna);
                LAUNCH(k_dt_transpose, tgT, tb, 0, s, sT, out, W, H);
            } else {
                LAUNCH(k_dt_cols, colBlocks, colThreads, 0, s, out, Dy, F, K, H, W, lna);
            }
        }
    } catch (...) {
        free_all(tmp, s);
        throw;
    }
    free_all(tmp, s);
}

static void backward_impl(fbs_system S, const float* g_dldx, const float* t, const float* c, float* dt, float* dc,
                          cudaStream_t s) {
    if (!S || !g_dldx || !t || !c || !dt || !dc) throw Err(FBS_EINVAL, "null pointer");
    fbs_grid g = S->g;
    pdl_break(s);
    const int64_t M = g->M;
    const int K = S->K;
    const size_t KM = (size_t)K * M;
    if (!S->xb) {
        S->xb = dalloc<float>(S->allocs, KM, s);
        S->u = dalloc<float>(S->allocs, KM, s);
        S->bwd = alloc_scalars(S->allocs, g->F * K, s);
    }
    CellGeom geo{g->F, g->H, g->W, g->ncx, g->ncy, g->colStart, g->rowStart};
    // u = S g (∂f/∂b = A⁻¹(S ∂f/∂x̂)), solved from x0 = 0 (reading #14)
    LAUNCH(k_splat<false>, grid_for(g->ncells * 32, 256, 1 << 20), 256, 0, s, geo, g->cellOff, g->heads, g->perm, nullptr, g_dldx, K,
           M, nullptr, S->u, S->inflags);
    VecArgs a = make_args(S, S->bwd, S->xb, S->u);
    S->rMasked = false;  // u = S g need not vanish on dead vertices: the lift reads w = mask∘r
    const VecArgs as = split_args(S, a);
    // k_assemble here only zeroes x and forms ‖u‖² (diag(A), μ0 are recomputed from the same inputs)
    LAUNCH(k_assemble, vec_blocks(as), kThreads, 0, s, as, S->diagA, S->mu0, FBS_INIT_ZERO, S->bwd);
    run_pcg(S, a, true, s);
    LAUNCH(k_bwd_finalize, grid_for(g->N), kThreads, 0, s, g->vid, S->xb, S->xh, c, t, M, K, g->F,
           (int64_t)g->H * g->W, dt, dc);
    S->has_backward = true;
}

// ===================================================================================== ABI
namespace fbs {
namespace {
int guard(const char* where, const std::function<void()>& body) {
    try {
        body();
        t_err.clear();
        return FBS_OK;
    } catch (const Err& e) {
        t_err = std::string(where) + ": " + e.what();
        return e.code;
    } catch (const std::exception& e) {
        t_err = std::string(where) + ": " + e.what();
        return FBS_ECUDA;
    } catch (...) {
        t_err = std::string(where) + ": unknown error";
        return FBS_ECUDA;
    }
}
}  // namespace
}  // namespace fbs

extern "C" {

void fbs_default_grid_opts(fbs_grid_opts* o) {
    if (!o) return;
    o->n_bistoch = 20;
    o->build_pyramid = 1;
    o->dims = 5;
}

void fbs_default_solve_opts(fbs_solve_opts* o) {
    if (!o) return;
    o->precond = FBS_PRECOND_HIER;
    o->init = FBS_INIT_HIER;
    o->mode = FBS_MODE_FIXED;
    o->iters = 25;
    o->tol = 1e-6;
    o->max_iters = 2000;
    o->precond_alpha = 2.0;
    o->precond_beta = 5.0;
    o->init_alpha = 4.0;
    o->init_beta = 0.0;
    o->lowrank_eps = 0.0;
}

int fbs_grid_build(const uint8_t* rgb, int frames, int height, int width, double sxy, double sl, double suv,
                   const fbs_grid_opts* opts, fbs_stream stream, fbs_grid* out) {
    return guard("fbs_grid_build", [&] {
        grid_build_impl(rgb, frames, height, width, sxy, sl, suv, opts, (cudaStream_t)stream, out);
    });
}

int fbs_grid_info(fbs_grid g, int64_t* n_pixels, int64_t* n_vertices, int* n_levels, int64_t* frame_vertices,
                  int64_t* level_vertices, int32_t* frame_levels) {
    return guard("fbs_grid_info", [&] {
        if (!g) throw Err(FBS_EINVAL, "null grid");
        if (n_pixels) *n_pixels = g->N;
        if (!n_vertices && !n_levels && !frame_vertices && !level_vertices && !frame_levels) return;
        ensure_sizes(g);  // the sizes are data-dependent: read back once (synchronises the grid's stream)
        if (n_vertices) *n_vertices = g->Mx;
        if (n_levels) *n_levels = g->Lx;
        if (frame_vertices)
            for (int f = 0; f < g->F; ++f) frame_vertices[f] = g->frameOffH[f + 1] - g->frameOffH[f];
        if (level_vertices)
            for (int k = 0; k < g->Lx; ++k) level_vertices[k] = g->levelMx[k];
        if (frame_levels)
            for (int f = 0; f < g->F; ++f) frame_levels[f] = g->frameLevelsH[f];
    });
}

int fbs_grid_export(fbs_grid g, uint64_t* keys, int32_t* vid, int32_t* nbr, int32_t* m, float* n, float* res) {
    return guard("fbs_grid_export", [&] {
        if (!g) throw Err(FBS_EINVAL, "null grid");
        ensure_sizes(g);
        cudaStream_t s = g->stream;
        const int64_t M = g->Mx;
        if (keys) ck(memcpy_async(keys, g->keys, M * 8, cudaMemcpyDeviceToHost, s), "d2h");
        if (vid) ck(memcpy_async(vid, g->vid, g->N * 4, cudaMemcpyDeviceToHost, s), "d2h");
        if (m) ck(memcpy_async(m, g->m, M * 4, cudaMemcpyDeviceToHost, s), "d2h");
        if (n) ck(memcpy_async(n, g->n, M * 4, cudaMemcpyDeviceToHost, s), "d2h");
        if (nbr) {
            AllocList tmp;
            int* d = dalloc<int>(tmp, (size_t)M * 10, s);
            LAUNCH(k_export_nbr, grid_for(M), kThreads, 0, s, g->nbr, (int)M, d);
            ck(memcpy_async(nbr, d, (size_t)M * 40, cudaMemcpyDeviceToHost, s), "d2h");
            free_all(tmp, s);
        }
        if (res) {
            if (g->bistoch_residual < 0.f) {  // reporting only: max|n∘B̄n − m| / max m, on request
                AllocList tmp;
                unsigned* d = dalloc<unsigned>(tmp, 2, s);
                zero_words(d, 2 * sizeof(unsigned), s);
                LAUNCH(k_bistoch_residual, grid_for(M), kThreads, 0, s, g->nbr, g->m, g->n, (int)M, d,
                       (float)(2 * g->dims));
                unsigned h2[2];
                ck(memcpy_async(h2, d, sizeof(h2), cudaMemcpyDeviceToHost, s), "d2h");
                ck(cudaStreamSynchronize(s), "sync");
                free_all(tmp, s);
                float e, mm;
                std::memcpy(&e, &h2[0], 4);
                std::memcpy(&mm, &h2[1], 4);
                g->bistoch_residual = (mm > 0.f) ? e / mm : 0.f;
            }
            *res = g->bistoch_residual;
        }
        ck(cudaStreamSynchronize(s), "sync");
    });
}

int fbs_pyramid_export(fbs_grid g, int level, uint64_t* keys, int32_t* parent, int32_t* count) {
    return guard("fbs_pyramid_export", [&] {
        if (!g) throw Err(FBS_EINVAL, "null grid");
        ensure_sizes(g);
        if (level < 1 || level >= g->Lx) throw Err(FBS_EINVAL, "level out of range");
        cudaStream_t s = g->stream;
        const Level& L = g->lv[level];
        const int64_t Mk = g->levelMx[level], Mprev = g->levelMx[level - 1];
        if (keys) ck(memcpy_async(keys, L.keys, Mk * 8, cudaMemcpyDeviceToHost, s), "d2h");
        if (parent) ck(memcpy_async(parent, L.parent, Mprev * 4, cudaMemcpyDeviceToHost, s), "d2h");
        if (count) ck(memcpy_async(count, L.count, Mk * 4, cudaMemcpyDeviceToHost, s), "d2h");
        ck(cudaStreamSynchronize(s), "sync");
    });
}

void fbs_grid_destroy(fbs_grid g) {
    if (!g) return;
    free_all(g->allocs, g->stream);
    for (auto& b : g->uploads) pinned_put(b, g->stream);
    delete g;
}

int fbs_solve(fbs_grid g, const float* t, int K, const float* c, double lam, const fbs_solve_opts* opts, float* x,
              float* y, fbs_system* sys_out, fbs_stream stream) {
    return guard("fbs_solve", [&] { solve_impl(g, t, K, c, lam, opts, x, y, sys_out, (cudaStream_t)stream); });
}

int fbs_solve_robust(fbs_grid g, const float* t, int K, const float* c_init, double lam, const fbs_solve_opts* opts,
                     double sigma_gm, int n_irls, float* x, float* c_out, fbs_stream stream) {
    return guard("fbs_solve_robust", [&] {
        robust_impl(g, t, K, c_init, lam, opts, sigma_gm, n_irls, x, c_out, (cudaStream_t)stream);
    });
}

int fbs_dt_filter(const uint8_t* rgb, int frames, int height, int width, const float* in, int K, double sigma_s,
                  double sigma_r, int n_iters, float* out, fbs_stream stream) {
    return guard("fbs_dt_filter", [&] {
        dt_impl(rgb, frames, height, width, in, K, sigma_s, sigma_r, n_iters, out, (cudaStream_t)stream);
    });
}

int fbs_solve_backward(fbs_system S, const float* dldx, const float* t, const float* c, float* dt, float* dc,
                       fbs_stream stream) {
    return guard("fbs_solve_backward", [&] { backward_impl(S, dldx, t, c, dt, dc, (cudaStream_t)stream); });
}

int fbs_system_stats(fbs_system S, int32_t* iters, double* relres, int32_t* bwd_iters, int32_t* status) {
    return guard("fbs_system_stats", [&] {
        if (!S) throw Err(FBS_EINVAL, "null system");
        cudaStream_t s = S->stream;
        const int FK = S->g->F * S->K;
        std::vector<double> rr(FK), bb(FK);
        std::vector<int> st(FK), st2(FK, 0);
        int inflags = 0;
        ck(memcpy_async(&inflags, S->inflags, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
        ck(memcpy_async(rr.data(), S->fwd.rr, FK * 8, cudaMemcpyDeviceToHost, s), "d2h");
        ck(memcpy_async(bb.data(), S->fwd.bb, FK * 8, cudaMemcpyDeviceToHost, s), "d2h");
        ck(memcpy_async(st.data(), S->fwd.status, FK * 4, cudaMemcpyDeviceToHost, s), "d2h");
        if (iters) ck(memcpy_async(iters, S->fwd.iters, FK * 4, cudaMemcpyDeviceToHost, s), "d2h");
        if (S->xb) {
            ck(memcpy_async(st2.data(), S->bwd.status, FK * 4, cudaMemcpyDeviceToHost, s), "d2h");
            if (bwd_iters) ck(memcpy_async(bwd_iters, S->bwd.iters, FK * 4, cudaMemcpyDeviceToHost, s), "d2h");
        } else if (bwd_iters) {
            for (int i = 0; i < FK; ++i) bwd_iters[i] = 0;
        }
        ck(cudaStreamSynchronize(s), "sync");
        if (relres)
            for (int i = 0; i < FK; ++i) relres[i] = bb[i] > 0 ? std::sqrt(rr[i] / bb[i]) : std::sqrt(rr[i]);
        if (status) {
            int acc = inflags;
            for (int i = 0; i < FK; ++i) acc |= st[i] | st2[i];
            *status = acc;
        }
    });
}

int fbs_system_export(fbs_system S, float* sc, float* b, float* diagA, float* y0, float* y, float* db) {
    return guard("fbs_system_export", [&] {
        if (!S) throw Err(FBS_EINVAL, "null system");
        fbs_grid g = S->g;
        ensure_sizes(g);
        cudaStream_t s = S->stream;
        const int64_t M = g->Mx;
        const int K = S->K;
        const size_t KM = (size_t)K * M;
        AllocList tmp;
        float* d = dalloc<float>(tmp, KM, s);
        auto vk = [&](const float* src, float* host) {
            LAUNCH(k_export_vk, grid_for(KM), kThreads, 0, s, src, nullptr, M, g->M, K, d);
            ck(memcpy_async(host, d, KM * 4, cudaMemcpyDeviceToHost, s), "d2h");
            ck(cudaStreamSynchronize(s), "sync");
        };
        if (sc) ck(memcpy_async(sc, S->sc, M * 4, cudaMemcpyDeviceToHost, s), "d2h");
        if (diagA) ck(memcpy_async(diagA, S->diagA, M * 4, cudaMemcpyDeviceToHost, s), "d2h");
        ck(cudaStreamSynchronize(s), "sync");
        if (b) vk(S->b, b);
        if (y0) vk(S->y0, y0);
        if (y) vk(S->xh, y);
        if (db) {
            if (S->xb) vk(S->xb, db);
            else std::memset(db, 0, KM * 4);
        }
        free_all(tmp, s);
        ck(cudaStreamSynchronize(s), "sync");
    });
}

void fbs_system_destroy(fbs_system S) {
    if (!S) return;
    free_all(S->allocs, S->stream);
    delete S;
}

int fbs_slice(fbs_grid g, const float* y, int K, float* x, fbs_stream stream) {
    return guard("fbs_slice", [&] {
        pdl_break((cudaStream_t)stream);
        if (!g || !y || !x) throw Err(FBS_EINVAL, "null pointer");
        if (K < 1 || K > kMaxK) throw Err(FBS_EINVAL, "K must be in [1, 64]");
        cudaStream_t s = (cudaStream_t)stream;
        slice(g, y, g->M, K, 0, x, s);
    });
}

int fbs_splat(fbs_grid g, const float* p, int K, float* out, fbs_stream stream) {
    return guard("fbs_splat", [&] {
        pdl_break((cudaStream_t)stream);
        if (!g || !p || !out) throw Err(FBS_EINVAL, "null pointer");
        if (K < 1 || K > kMaxK) throw Err(FBS_EINVAL, "K must be in [1, 64]");
        cudaStream_t s = (cudaStream_t)stream;
        AllocList tmp;
        const size_t KM = (size_t)K * g->M;
        float* planar = dalloc<float>(tmp, KM, s);
        CellGeom geo{g->F, g->H, g->W, g->ncx, g->ncy, g->colStart, g->rowStart};
        LAUNCH(k_splat<false>, grid_for(g->ncells * 32, 256, 1 << 20), 256, 0, s, geo, g->cellOff, g->heads, g->perm, nullptr, p, K,
               g->M, nullptr, planar, nullptr);
        LAUNCH(k_export_vk, grid_for(KM), kThreads, 0, s, planar, g->frameOff + g->F, (int64_t)0, g->M, K, out);
        free_all(tmp, s);
    });
}

int fbs_blur(fbs_grid g, const float* v, float* out, fbs_stream stream) {
    return guard("fbs_blur", [&] {
        pdl_break((cudaStream_t)stream);
        if (!g || !v || !out) throw Err(FBS_EINVAL, "null pointer");
        ensure_sizes(g);  // the caller's vectors hold exactly M vertices
        LAUNCH(k_blur, grid_for(g->Mx), kThreads, 0, (cudaStream_t)stream, g->nbr, v, g->Mx, (float)(2 * g->dims), out);
    });
}

int fbs_system_apply_A(fbs_system S, const float* y, float* out, fbs_stream stream) {
    return guard("fbs_system_apply_A", [&] {
        pdl_break((cudaStream_t)stream);
        if (!S || !y || !out) throw Err(FBS_EINVAL, "null pointer");
        cudaStream_t s = (cudaStream_t)stream;
        fbs_grid g = S->g;
        ensure_sizes(g);
        AllocList tmp;
        const size_t KM = (size_t)S->K * g->M;
        float* ys = dalloc<float>(tmp, KM, s);
        LAUNCH(k_import_vk, grid_for((size_t)S->K * g->Mx), kThreads, 0, s, y, nullptr, g->Mx, g->M, S->K, ys);
        VecArgs a = make_args(S, S->fwd, S->xh, S->b);
        LAUNCH(k_apply_A, grid_for(g->M), kThreads, 0, s, a, ys, out);
        free_all(tmp, s);
    });
}

int fbs_system_apply_precond(fbs_system S, const float* r, float* out, fbs_stream stream) {
    return guard("fbs_system_apply_precond", [&] {
        pdl_break((cudaStream_t)stream);
        if (!S || !r || !out) throw Err(FBS_EINVAL, "null pointer");
        cudaStream_t s = (cudaStream_t)stream;
        fbs_grid g = S->g;
        ensure_sizes(g);
        AllocList tmp;
        const size_t KM = (size_t)S->K * g->M;
        float* w = dalloc<float>(tmp, KM, s);
        zero_words(w, KM * sizeof(float), s);
        LAUNCH(k_import_vk, grid_for((size_t)S->K * g->Mx), kThreads, 0, s, r, S->mu0, g->Mx, g->M, S->K, w);
        if (S->useHierP) {
            float* planar = dalloc<float>(tmp, KM, s);
            HierArgs h = S->hP;
            VecArgs a = make_args(S, S->fwd, S->xh, S->b);
            tree_lift<HIER_PLAIN>(S, h, w, s);
            tree_coarse<HIER_PLAIN>(S, h, a, 0, s);
            tree_level0<HIER_PLAIN>(S, h, a, w, planar, 0, s);
            LAUNCH(k_export_vk, grid_for(KM), kThreads, 0, s, planar, nullptr, g->Mx, g->M, S->K, out);
        } else {
            LAUNCH(k_precond_out, grid_for(g->Mx), kThreads, 0, s, w, S->mu0, nullptr, nullptr, 0, g->Mx, g->M, S->K, out);
        }
        free_all(tmp, s);
    });
}

const char* fbs_last_error(void) { return t_err.c_str(); }
int fbs_version(void) { return 1; }

int fbs_set_allocator(const fbs_allocator* a) {
    return guard("fbs_set_allocator", [&] {
        if (a && (!a->alloc || !a->free)) throw Err(FBS_EINVAL, "allocator needs both alloc and free");
        std::lock_guard<std::mutex> lk(g_alloc_mu);
        g_allocator = a ? *a : fbs_allocator{};
    });
}
int64_t fbs_launch_count(void) { return (int64_t)g_launches.load(); }

int fbs_profile_enable(int on) {
    fbs::g_prof_on.store(on ? 1 : 0);
    return FBS_OK;
}

int fbs_profile_reset(void) {
    return guard("fbs_profile_reset", [&] {
        std::lock_guard<std::mutex> lk(fbs::g_prof_mu);
        for (auto& r : fbs::g_prof) {
            fbs::g_ev_pool.push_back(r.a);
            fbs::g_ev_pool.push_back(r.b);
        }
        fbs::g_prof.clear();
    });
}

int fbs_profile_report(char* buf, size_t len) {
    std::string js;
    int rc = guard("fbs_profile_report", [&] {
        std::lock_guard<std::mutex> lk(fbs::g_prof_mu);
        std::map<std::string, std::pair<long long, double>> acc;
        for (auto& r : fbs::g_prof) {
            ck(cudaEventSynchronize(r.b), "cudaEventSynchronize");
            float ms = 0.f;
            ck(cudaEventElapsedTime(&ms, r.a, r.b), "cudaEventElapsedTime");
            auto& e = acc[r.name];
            e.first += 1;
            e.second += ms;
        }
        // FBS_TIMELINE=<path>: every profiled launch as CSV (name, stream, start, duration in µs
        // relative to the first one) for overlap analysis
        if (const char* tl = std::getenv("FBS_TIMELINE")) {
            if (FILE* fh = std::fopen(tl, "w")) {
                std::fprintf(fh, "name,stream,start_us,dur_us\n");
                for (auto& r : fbs::g_prof) {
                    float t0 = 0.f, d = 0.f;
                    cudaEventElapsedTime(&t0, fbs::g_prof.front().a, r.a);
                    cudaEventElapsedTime(&d, r.a, r.b);
                    std::fprintf(fh, "%s,%p,%.3f,%.3f\n", r.name, (void*)r.s, 1e3 * t0, 1e3 * d);
                }
                std::fclose(fh);
            }
        }
        js = "{";
        bool first = true;
        for (auto& kv : acc) {
            char tmp[256];
            std::snprintf(tmp, sizeof(tmp), "%s\"%s\": [%lld, %.6f]", first ? "" : ", ", kv.first.c_str(),
                          kv.second.first, kv.second.second);
            js += tmp;
            first = false;
        }
        js += "}";
    });
    if (rc != FBS_OK) return -rc;
    if (buf && len > 0) {
        std::strncpy(buf, js.c_str(), len - 1);
        buf[len - 1] = 0;
    }
    return (int)js.size() + 1;
}

}  // extern "C"
