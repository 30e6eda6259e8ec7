/*
 * fbs.h — C ABI of the B200-native bilateral-space solve
 *         (Fast Bilateral Solver, Barron & Poole, arXiv 1511.03296).
 *
 * The library implements the hot path of the paper's method on sm_100a:
 *   grid build      simplified bilateral grid            PAPER.md:114-116 (Sec. 2, Eq. equiv)
 *   bistochastize   Alg. 1                               PAPER.md:656-672 (Supp. Sec. 1)
 *   assemble        A = λ(Dm − Dn B̄ Dn) + diag(Sc), b = S(c∘t)   PAPER.md:124-127 (Eq. quad_min)
 *   precondition    Jacobi / hierarchical                PAPER.md:227-285 (Sec. 4, Eq. hier_precond)
 *   initialise      flat / hierarchical                  PAPER.md:238-241, 287-293 (Eq. flat_init)
 *   solve           PCG, Alg. 2                          PAPER.md:710-742 (Supp. Sec. 1)
 *   slice           x̂ = Sᵀ ŷ                             PAPER.md:137-140 (Eq. solution)
 *   backward        ∂f/∂t, ∂f/∂c by one more solve       PAPER.md:191-201 (Sec. 3)
 * Readings of the paper where it is silent or ambiguous are numbered in DESIGN.md §3: #1..#19
 * follow SURVEY.md §8(c); #20..#29 are this build's own and change what the kernels compute:
 * #20 difference-form A, #21 σxy cell limit, #22 pyramid cell capacity, #23 ρ from the lift,
 * #24 coarse lifts as prefix differences, #25 robust objective, #26 low-rank row selection,
 * #27 D = 3 grid, #28 domain-transform filter, #29 fixed-count parity on unstable iterates.
 *
 * Conventions (all entry points)
 *   - Every pointer argument named *_dev is DEVICE memory owned by the caller and only
 *     borrowed for the enqueued work; pointers named *_host are HOST memory.
 *   - Work is enqueued on `stream` (a cudaStream_t; NULL = legacy default stream).  The
 *     compute calls only enqueue: fbs_grid_build sizes its buffers by capacities known on the
 *     host (vertices ≤ pixels, pyramid level k ≤ min(level k−1, cells_k × codes_k)) and its
 *     kernels read the data-dependent counts on the device, so grid build + FIXED-mode solve
 *     (+ slice, backward, low-rank) can be captured into a CUDA graph and replayed.  The
 *     exceptions are stated per call: TOL-mode solves poll the device's active count from the
 *     host unless the stream is capturing (then a device-side loop is captured) or the solve is
 *     a Jacobi one on frames of ≤ 262144 pixels (one launch, fbs_solve); the query and
 *     export calls (fbs_grid_info, *_export, *_stats) synchronise.
 *   - Layouts: RGB is interleaved uint8 [frames][H][W][3]; pixel vectors are planar float
 *     [frames][K][H][W] (pixel p = y·W + x); confidences float [frames][H][W];
 *     vertex vectors are float [M][K] in CANONICAL vertex order: ascending packed key
 *     frame(8)‖by(16)‖bx(16)‖bl(8)‖bu(8)‖bv(8) (reading #3), frames concatenated.
 *   - Return value: FBS_OK (0) or an FBS_E* code; fbs_last_error() gives a thread-local
 *     message.  Data-dependent outcomes (breakdown, non-convergence) are reported by
 *     fbs_system_stats after the stream has been synchronised.  No exception crosses
 *     the ABI.  There is no CPU fallback: without a CUDA device every call fails with
 *     FBS_ECUDA.
 *   - Handles own their internal device buffers (one stream-ordered arena per handle, from the
 *     device's default memory pool or a caller allocator) and release them in *_destroy, which
 *     enqueues the frees on the stream the handle was created on.
 *   - Thread safety: a built grid is immutable; concurrent fbs_solve calls on distinct
 *     streams with distinct outputs are allowed.  A system handle must not be used by
 *     two streams at once.
 */
#ifndef FBS_H
#define FBS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* fbs_stream; /* == cudaStream_t */
typedef struct fbs_grid_s* fbs_grid;
typedef struct fbs_system_s* fbs_system;

/* ---------------------------------------------------------------- status codes */
#define FBS_OK 0
#define FBS_EINVAL 1 /* bad argument (see each call)                                   */
#define FBS_ENOMEM 2 /* device allocation failed                                       */
#define FBS_ECUDA 3  /* CUDA runtime error (message in fbs_last_error)                 */
#define FBS_ELIMIT 4 /* structural limit exceeded: a σxy cell holds > 64 pixels        */
                     /* (reading #21)                                    */
#define FBS_ESTATE 5 /* handle used in the wrong state (e.g. backward before forward)  */

/* bits of the `status` word returned by fbs_system_stats */
#define FBS_ST_BREAKDOWN 1     /* a (frame, channel) stopped on ρ = 0 or dᵀq ≤ 0 (reading #11) */
#define FBS_ST_NOTCONVERGED 2  /* TOL mode: max_iters reached before ‖r‖ ≤ tol‖b‖           */
#define FBS_ST_NEG_CONF 4      /* some confidence c < 0 (the paper requires c ≥ 0) */
#define FBS_ST_NONFINITE 8     /* a non-finite c, t (forward) or dL/dx (backward) entered S      */

/* ---------------------------------------------------------------- options */
typedef struct {
    int n_bistoch;     /* Alg. 1 iterations, fixed count (reading #5); default 20          */
    int build_pyramid; /* 1: build the Supp. Sec. 2 pyramid (needed by HIER precond/init) */
    int dims;          /* D: 5 = XYLUV grid (default); 3 = XYL grid of a grayscale reference */
                       /* (chroma not used, B̄ = 2·3·I + Adj, reading #27)     */
} fbs_grid_opts;

enum { FBS_PRECOND_JACOBI = 0, FBS_PRECOND_HIER = 1 };
enum { FBS_INIT_FLAT = 0, FBS_INIT_HIER = 1, FBS_INIT_ZERO = 2 };
enum { FBS_MODE_FIXED = 0, FBS_MODE_TOL = 1 };

typedef struct {
    int precond;          /* FBS_PRECOND_*; default HIER                          */
    int init;             /* FBS_INIT_*; default HIER                              */
    int mode;             /* FBS_MODE_FIXED: exactly `iters` iterations (Alg. 2);   */
                          /* FBS_MODE_TOL: stop when ‖r_i‖₂ ≤ tol·‖b‖₂ (recurrence residual,     */
                          /* tested before every iteration incl. i = 0, reading #11)            */
    int iters;            /* FIXED iteration count; default 25                    */
    double tol;           /* TOL relative residual; default 1e-6                                 */
    int max_iters;        /* TOL cap; default 2000                                               */
    double precond_alpha; /* z_weight α, β of the preconditioner; default 2, 5    */
    double precond_beta;
    double init_alpha;    /* z_weight α, β of the initialisation; default 4, 0    */
    double init_beta;
    double lowrank_eps;   /* > 0 (K > 1): low-rank reduction of the right-hand sides (Supp. §4,  */
                          /* PAPER.md:867-900): solve only the rows of R' holding ≥ (1 − ε) of  */
                          /* the mass, Y = (A⁻¹Q̃)R̃ (reading #26); 0 = off (default)            */
} fbs_solve_opts;

/* ---------------------------------------------------------------- device memory
 * Handles allocate their internal buffers stream-ordered on the stream they are created on.
 * By default that is cudaMallocAsync / cudaFreeAsync on the device's default memory pool; a
 * caller may route them through its own allocator (e.g. PyTorch's caching allocator):
 *   alloc(bytes, ctx, stream) → device pointer usable in stream order on `stream` (NULL: fails
 *                               the call with FBS_ENOMEM);
 *   free(ptr, ctx, stream)    → release; all work the library enqueued on its buffers is
 *                               ordered on `stream` before this point.
 * fbs_set_allocator applies to handles created afterwards (a handle keeps the allocator it was
 * created with and calls its free when destroyed, so the callbacks must stay valid until then);
 * NULL restores the default.  Returned pointers must be 16-byte aligned (vector loads and bulk
 * copies; FBS_EINVAL otherwise).  Not thread-safe against concurrent handle creation. */
typedef struct {
    void* (*alloc)(size_t bytes, void* ctx, fbs_stream stream);
    void (*free)(void* ptr, void* ctx, fbs_stream stream);
    void* ctx;
} fbs_allocator;
int fbs_set_allocator(const fbs_allocator* a);

void fbs_default_grid_opts(fbs_grid_opts* o);
void fbs_default_solve_opts(fbs_solve_opts* o);

/* ---------------------------------------------------------------- grid */
/* Build the simplified bilateral grid of `frames` independent reference images.
 *   rgb_dev   uint8 [frames][height][width][3], device.
 *   sigma_*   bandwidths of Eq. bilateral_affinity.  Pixel (x, y) with
 *             integer luma/chroma numerators Yn,Un,Vn (reading #1) maps to the vertex
 *             (⌊x/σxy⌋, ⌊y/σxy⌋, ⌊Yn/256σl⌋, ⌊Un/256σuv⌋, ⌊Vn/256σuv⌋), each one IEEE
 *             fp64 division then floor (reading #2).
 * Then runs opts->n_bistoch iterations of Alg. 1 and (if opts->build_pyramid) builds the
 * pyramid of PAPER.md:745-766 (reading #8).  Enqueue-only (no host synchronisation): buffers
 * are sized by capacities (memory ≈ 200 B per pixel with the pyramid), counts live on the device.
 * Errors: FBS_EINVAL if a pointer is NULL, frames ∉ [1, 256], height or width ∉
 * [1, 65535·σxy], σl < 1 or σuv < 1 (8-bit key fields), σxy < 1, or σxy > 8: a σxy cell is one
 * warp of ≤ 64 pixels (reading #21; every setting of the paper uses σxy ≤ 8, PAPER.md:433, :515,
 * :974); FBS_ENOMEM; FBS_ECUDA.  The build's internal invariant checks (FBS_ELIMIT, FBS_ECUDA)
 * are reported by the first synchronous query (fbs_grid_info / fbs_grid_export). */
int fbs_grid_build(const uint8_t* rgb_dev, int frames, int height, int width, double sigma_xy,
                   double sigma_l, double sigma_uv, const fbs_grid_opts* opts, fbs_stream stream,
                   fbs_grid* out);

/* Sizes of a built grid (host outputs; any pointer may be NULL).  The counts are data-dependent
 * and computed on the device: the first call that asks for more than n_pixels synchronises the
 * grid's stream once (the values are cached with the grid).
 *   frame_vertices_host  int64 [frames]      vertices per frame
 *   level_vertices_host  int64 [n_levels]    Σ over frames of level-k vertex counts
 *   frame_levels_host    int32 [frames]      pyramid levels of each frame (until 1 vertex) */
int fbs_grid_info(fbs_grid g, int64_t* n_pixels, int64_t* n_vertices, int* n_levels,
                  int64_t* frame_vertices_host, int64_t* level_vertices_host,
                  int32_t* frame_levels_host);

/* Copy the grid to host memory in canonical order (synchronous; any pointer may be NULL).
 *   keys_host  uint64 [M]      packed keys (reading #3), strictly ascending
 *   vid_host   int32  [N]      vertex of each pixel (S as a hard assignment)
 *   nbr_host   int32  [M][10]  ±1 neighbours, slots (x−,x+,y−,y+,l−,l+,u−,u+,v−,v+), −1 absent
 *   m_host     int32  [M]      splat counts m = S1
 *   n_host     float  [M]      Alg. 1 result n (Dn = diag(n))
 *   bistoch_residual_host      max|n∘B̄n − m| / max m after the last Alg. 1 step */
int fbs_grid_export(fbs_grid g, uint64_t* keys_host, int32_t* vid_host, int32_t* nbr_host,
                    int32_t* m_host, float* n_host, float* bistoch_residual_host);

/* Pyramid level `level` ≥ 1 in canonical order (synchronous):
 *   keys_host    uint64 [M_level]       level keys (fields halved `level` times)
 *   parent_host  int32  [M_{level−1}]   parent (in level) of each level−1 vertex = S_{level−1}
 *   count_host   int32  [M_level]       P(1): level-0 vertices under each level vertex */
int fbs_pyramid_export(fbs_grid g, int level, uint64_t* keys_host, int32_t* parent_host,
                       int32_t* count_host);

void fbs_grid_destroy(fbs_grid g);

/* ---------------------------------------------------------------- solve */
/* Solve A y = b for K channels sharing one A (reading #13) and slice.
 *   t_dev      float [frames][K][H][W]   targets
 *   c_dev      float [frames][H][W]      confidences, ≥ 0 (c < 0 and non-finite c, t are flagged in
 *                                        the status bits FBS_ST_NEG_CONF / FBS_ST_NONFINITE)
 *   lambda     > 0                       smoothness weight λ
 *   x_dev      float [frames][K][H][W]   output x̂ = Sᵀŷ (may alias nothing else)
 *   y_dev      float [M][K] or NULL      bilateral-space solution ŷ
 *   sys_out    receives the system handle (A-state, M⁻¹, ŷ) for fbs_solve_backward and
 *              the stats/export calls; NULL = destroy it after the solve.
 * Each (frame, channel) runs its own PCG scalars and stopping rule (reading #13).  The frames are
 * split into groups whose PCGs run concurrently on side streams forked from and joined to
 * `stream` (they are independent systems); FIXED mode only enqueues work, TOL mode polls each
 * group's active count from the host one chunk (6 iterations, fewer near the predicted stopping
 * point) behind and returns when all have stopped; when `stream` is being captured into a CUDA
 * graph it adds a conditional while node instead (device-side loop, no host polls, replayable);
 * FBS_TOL_GRAPH=1 runs such a loop as its own graph per solve.  Jacobi solves of frames of
 * ≤ 8192 pixels (FBS_SMALL_PX) run each (frame, channel)'s whole PCG in one CTA instead, and of
 * ≤ 98304 pixels (≤ 262144 with ≥ 16 (frame, channel)s; FBS_CLUSTER_PX) in one cluster of 8
 * CTAs: one launch, in either mode enqueue-only (the stopping rule is decided on the device).
 * opts->lowrank_eps > 0 with K > 1 reduces B per frame first (Supp. §4): the reduced solve
 * carries K channels of which those at or above the frame's kept rank t_f have zero right-hand
 * sides and retire at iteration 0 (no host synchronisation); sys_out must then be NULL.
 * Errors: FBS_EINVAL (NULL pointer, K ∉ [1, 64], λ ≤ 0 or not finite, HIER precond/init
 * on a grid built without pyramid, bad opts); FBS_ENOMEM; FBS_ECUDA. */
int fbs_solve(fbs_grid g, const float* t_dev, int K, const float* c_dev, double lambda,
              const fbs_solve_opts* opts, float* x_dev, float* y_dev, fbs_system* sys_out,
              fbs_stream stream);

/* Robust bilateral solver (Supp. §3, Alg. 3 "The Geman-McClure Robust Bilateral Solver",
 * PAPER.md:798-813):  c ← c_init;  n_irls times:  x̂ ← solve(t, c);  e ← x̂ − t;
 * c ← 2σ_gm² / (σ_gm² + e∘e)².  Every inner solve is fbs_solve with `opts` on the same grid
 * (n, pyramid and the smoothness part of A are reused; only diag(S c) and b change).
 *   t_dev       float [frames][1][H][W]   scalar targets (K = 1, reading #25)
 *   c_init_dev  float [frames][H][W]      initial confidences, ≥ 0 (read only)
 *   sigma_gm    > 0                        Geman–McClure scale
 *   n_irls      ≥ 1                        IRLS iterations (the paper uses 32)
 *   x_dev       float [frames][1][H][W]   output: x̂ of the last inner solve
 *   c_out_dev   float [frames][H][W] or NULL   the weights after the last update (line 5)
 * Errors: as fbs_solve, plus FBS_EINVAL for K ≠ 1, σ_gm ≤ 0 or n_irls < 1. */
int fbs_solve_robust(fbs_grid g, const float* t_dev, int K, const float* c_init_dev, double lambda,
                     const fbs_solve_opts* opts, double sigma_gm, int n_irls, float* x_dev,
                     float* c_out_dev, fbs_stream stream);

/* Domain-transform post-filter of solver output ("post-processed by the domain
 * transform … included in all runtimes", :333 σ'_xy, σ'_rgb): the recursive-filter variant of
 * Gastal & Oliveira 2011, restated in reading #28 — n_iters (default 3) row + column passes with
 * per-pass σ_i = σ_s √3 2^(N−i)/√(4^N − 1), weights a_i^(1 + σ_s/σ_r Σ_c|ΔI_c|) from the RGB guide.
 *   rgb_dev  uint8 [frames][H][W][3]   guide (the reference image)
 *   in_dev   float [frames][K][H][W]   signal (e.g. fbs_solve's x)
 *   out_dev  float [frames][K][H][W]   output; may equal in_dev (in place)
 * Errors: FBS_EINVAL (NULL pointer, K ∉ [1, 64], σ ≤ 0, n_iters < 1, H or W > 16384); FBS_ENOMEM;
 * FBS_ECUDA. */
int fbs_dt_filter(const uint8_t* rgb_dev, int frames, int height, int width, const float* in_dev, int K,
                  double sigma_s, double sigma_r, int n_iters, float* out_dev, fbs_stream stream);

/* Backward pass: given g = ∂f/∂x̂ [frames][K][H][W], solve A d = S g
 * with the forward's preconditioner and stopping rule from d = 0 (reading #14), then
 *   ∂f/∂t = c ∘ Sᵀd              → dt_dev float [frames][K][H][W]
 *   ∂f/∂c = Σ_k Sᵀ(−d_k∘ŷ_k) + (Sᵀd_k)∘t_k   → dc_dev float [frames][H][W] (reading #15)
 * t_dev and c_dev must be the same arrays (unchanged) that were passed to fbs_solve. */
int fbs_solve_backward(fbs_system sys, const float* dldx_dev, const float* t_dev,
                       const float* c_dev, float* dt_dev, float* dc_dev, fbs_stream stream);

/* Per-(frame, channel) results (host outputs, synchronous; any pointer may be NULL):
 *   iterations_host   int32  [frames*K]  PCG iterations run (forward)
 *   relres_host       double [frames*K]  recurrence ‖r‖₂/‖b‖₂ at exit (forward)
 *   bwd_iterations_host int32 [frames*K] iterations of the last backward solve
 *   status_host       FBS_ST_* bits */
int fbs_system_stats(fbs_system sys, int32_t* iterations_host, double* relres_host,
                     int32_t* bwd_iterations_host, int32_t* status_host);

/* Copy the assembled system to host memory (synchronous; any pointer may be NULL):
 *   sc_host [M]  S c;   b_host [M][K]  S(c∘t);   diagA_host [M]  diag(A);
 *   y0_host [M][K]  initial state;   y_host [M][K]  solution ŷ;
 *   db_host [M][K]  ∂f/∂b of the last backward (zeros before any backward). */
int fbs_system_export(fbs_system sys, float* sc_host, float* b_host, float* diagA_host,
                      float* y0_host, float* y_host, float* db_host);

void fbs_system_destroy(fbs_system sys);

/* ---------------------------------------------------------------- operators (device, async)
 * fbs_blur and the fbs_system_apply_* hooks take caller vectors of exactly M vertices: their
 * first use on a grid reads M back (one synchronisation, as fbs_grid_info). */
/* x̂ = Sᵀy: y_dev float [M][K] canonical → x_dev float [frames][K][H][W]. */
int fbs_slice(fbs_grid g, const float* y_dev, int K, float* x_dev, fbs_stream stream);
/* out = S p: p_dev float [frames][K][H][W] → out_dev float [M][K]. */
int fbs_splat(fbs_grid g, const float* p_dev, int K, float* out_dev, fbs_stream stream);
/* out = B̄ v: v_dev, out_dev float [M] (reading #4). */
int fbs_blur(fbs_grid g, const float* v_dev, float* out_dev, fbs_stream stream);
/* out = A y and out = M⁻¹ r for the system's A and preconditioner; float [M][K]. */
int fbs_system_apply_A(fbs_system sys, const float* y_dev, float* out_dev, fbs_stream stream);
int fbs_system_apply_precond(fbs_system sys, const float* r_dev, float* out_dev,
                             fbs_stream stream);

/* ---------------------------------------------------------------- misc */
const char* fbs_last_error(void);
int fbs_version(void);
/* Number of CUDA kernels this library has launched in this process (monotone counter). */
int64_t fbs_launch_count(void);

/* Per-kernel device timing.  While enabled, every launch is bracketed by two CUDA events
 * recorded on its own stream.  fbs_profile_report synchronises those events and writes a JSON
 * object {"<kernel>": [launches, total_ms], ...} into buf (NUL-terminated, truncated to len);
 * it returns the number of bytes needed.  fbs_profile_reset clears the records. */
int fbs_profile_enable(int on);
int fbs_profile_report(char* buf, size_t len);
int fbs_profile_reset(void);

#ifdef __cplusplus
}
#endif
#endif /* FBS_H */
