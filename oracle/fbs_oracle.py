"""ORACLE (test infrastructure only) — fp64 CPU bilateral-space solve.

Every function follows a passage of PAPER.md (cited as ``PAPER.md:<line>``,
section / equation label / algorithm) or a reading listed in DESIGN.md §3
("Readings of the paper", numbered as in SURVEY.md §8(c)).  Library
primitives used as single steps: ``np.unique`` (the set of occupied grid
coordinates), ``np.searchsorted`` (looking a coordinate tuple up), scipy
sparse matrix products (S, B̄, A applied to vectors) and dense LAPACK solves in
the brute-force helpers.  Nothing is blocked, fused or reordered beyond what
the paper's definitions state.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg may import this module.  It shares no code with paper_1511_03296_b200/.

Parity pins: every public function is pinned by tests/test_oracle.py against
closed forms, worked examples (tests/golden/), brute force or invariants —
see DESIGN.md §4.  No function here is "parity unpinned".
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np
import scipy.sparse as sp
import scipy.sparse.csgraph  # noqa: F401  (connected components, reading #7)

D = 5  # dimensionality of XYLUV bilateral space (Supp §2: "m by 5 matrix")
BBAR_DIAG = 2 * D  # B̄ = Σ_d [1 2 1] along dim d → constant diagonal 2D (reading #4)

# Neighbour slot order (reading #3): (x−, x+, y−, y+, l−, l+, u−, u+, v−, v+).
# Vertex tuple columns: (frame, by, bx, bl, bu, bv).
COL = {"f": 0, "y": 1, "x": 2, "l": 3, "u": 4, "v": 5}
SLOT_DIMS = ("x", "y", "l", "u", "v")


# ----------------------------------------------------------------------------- grid
def yuv_numerators(rgb: np.ndarray):
    """Reading #1 (PAPER.md:94 "in the YUV colorspace", :103 p = (x, y, l, u, v)).

    BT.601 full range with 8-bit fixed-point coefficients, kept as exact
    integers:  l = Yn/256, u = Un/256, v = Vn/256 with
        Yn = 77R + 150G + 29B,  Un = −43R − 85G + 128B + 32768,
        Vn = 128R − 107G − 21B + 32768.
    """
    r = rgb[..., 0].astype(np.int64)
    g = rgb[..., 1].astype(np.int64)
    b = rgb[..., 2].astype(np.int64)
    Yn = 77 * r + 150 * g + 29 * b
    Un = -43 * r - 85 * g + 128 * b + 32768
    Vn = 128 * r - 107 * g - 21 * b + 32768
    return Yn, Un, Vn


def pixel_coords(rgb: np.ndarray, sigma_xy: float, sigma_l: float, sigma_uv: float) -> np.ndarray:
    """Quantised XYLUV coordinate of every pixel (PAPER.md:94-104 Eq. bilateral_affinity
    bandwidths; reading #2: floor of one IEEE fp64 division, origin 0, no offset).

    rgb: uint8 [F][H][W][3].  Returns int64 [F*H*W][6] = (frame, by, bx, bl, bu, bv)
    in row-major pixel order p = (f·H + y)·W + x.
    """
    F, H, W, _ = rgb.shape
    Yn, Un, Vn = yuv_numerators(rgb)
    fr, ys, xs = np.meshgrid(np.arange(F), np.arange(H), np.arange(W), indexing="ij")
    out = np.empty((F * H * W, 6), np.int64)
    out[:, 0] = fr.ravel()
    out[:, 1] = np.floor(ys.ravel().astype(np.float64) / np.float64(sigma_xy))
    out[:, 2] = np.floor(xs.ravel().astype(np.float64) / np.float64(sigma_xy))
    out[:, 3] = np.floor(Yn.ravel().astype(np.float64) / (256.0 * np.float64(sigma_l)))
    out[:, 4] = np.floor(Un.ravel().astype(np.float64) / (256.0 * np.float64(sigma_uv)))
    out[:, 5] = np.floor(Vn.ravel().astype(np.float64) / (256.0 * np.float64(sigma_uv)))
    return out


def pack_key(V: np.ndarray) -> np.ndarray:
    """Reading #3 key layout: frame(8) ‖ by(16) ‖ bx(16) ‖ bl(8) ‖ bu(8) ‖ bv(8), bits 63…0."""
    V = V.astype(np.uint64)
    return ((V[:, 0] << np.uint64(56)) | (V[:, 1] << np.uint64(40)) | (V[:, 2] << np.uint64(24))
            | (V[:, 3] << np.uint64(16)) | (V[:, 4] << np.uint64(8)) | V[:, 5])


@dataclass
class Grid:
    """Simplified bilateral grid (PAPER.md:114 "simplified bilateral grid", :111 S, :664 m = S1)."""

    V: np.ndarray  # int64 [M][6] vertex coordinates, canonical (ascending key) order
    vid: np.ndarray  # int64 [N] vertex of each pixel (hard assignment = S)
    m: np.ndarray  # int64 [M] splat counts m = S 1
    nbr: np.ndarray  # int64 [M][10] ±1 neighbours per dim, −1 if absent
    frames: int
    frame_start: np.ndarray  # int64 [F+1] first vertex of each frame
    dims: int = 5  # D: 5 = XYLUV (colour), 3 = XYL (grayscale reference, reading #27)

    @property
    def M(self) -> int:
        return self.V.shape[0]

    @property
    def N(self) -> int:
        return self.vid.shape[0]

    @property
    def keys(self) -> np.ndarray:
        return pack_key(self.V)


def _tuple_codes(V: np.ndarray) -> np.ndarray:
    """Injective int64 code of (by, bx, bl, bu, bv) with one guard value below and above each
    field (fields shifted by +1, widths 18/18/9/9/9 bits), so that ±1 in any field can never
    carry into a neighbouring field.  Used only to look tuples up (reading #3 order is not
    needed here; per-frame lookups are done on frame-restricted arrays)."""
    c = V[:, 1] + 1
    c = c * (1 << 18) + (V[:, 2] + 1)
    c = c * (1 << 9) + (V[:, 3] + 1)
    c = c * (1 << 9) + (V[:, 4] + 1)
    c = c * (1 << 9) + (V[:, 5] + 1)
    return c


def find_neighbours(V: np.ndarray) -> np.ndarray:
    """nbr[v][2d+s] = index of the tuple V[v] ± e_d (same frame), else −1.

    The structure of B̄ (PAPER.md:233, :107-112 Eq. factorization): each vertex
    is linked to its ±1 neighbours along each of the 5 dims (reading #4)."""
    M = V.shape[0]
    nbr = -np.ones((M, 2 * D), np.int64)
    for f in np.unique(V[:, 0]):
        idx = np.nonzero(V[:, 0] == f)[0]
        codes = _tuple_codes(V[idx])
        order = np.argsort(codes, kind="stable")
        sc = codes[order]
        for d, name in enumerate(SLOT_DIMS):
            for s, step in enumerate((-1, +1)):
                W2 = V[idx].copy()
                W2[:, COL[name]] += step
                q = _tuple_codes(W2)
                pos = np.searchsorted(sc, q)
                pos_c = np.minimum(pos, len(sc) - 1)
                hit = (pos < len(sc)) & (sc[pos_c] == q)
                nbr[idx[hit], 2 * d + s] = idx[order[pos_c[hit]]]
    return nbr


def build_grid(rgb: np.ndarray, sigma_xy: float, sigma_l: float, sigma_uv: float, dims: int = 5) -> Grid:
    """Simplified bilateral grid: unique occupied coordinates, hard splat map, counts,
    neighbours (PAPER.md:114-116 Eq. equiv, :664 m ← S1; readings #2, #3).
    dims = 3: the XYL grid of a grayscale reference (reading #27): the chroma
    coordinates are not used (held at 0)."""
    assert dims in (3, 5)
    F = rgb.shape[0]
    P = pixel_coords(rgb, sigma_xy, sigma_l, sigma_uv)
    if dims == 3:
        P[:, COL["u"]] = 0
        P[:, COL["v"]] = 0
    # np.unique(axis=0) sorts rows lexicographically by (frame, by, bx, bl, bu, bv)
    # = ascending packed key (reading #3 canonical order).
    V, vid, m = np.unique(P, axis=0, return_inverse=True, return_counts=True)
    vid = vid.reshape(-1)
    frame_start = np.searchsorted(V[:, 0], np.arange(F + 1))
    return Grid(V=V, vid=vid.astype(np.int64), m=m.astype(np.int64), nbr=find_neighbours(V),
                frames=F, frame_start=frame_start.astype(np.int64), dims=dims)


def splat_matrix(vid: np.ndarray, M: int) -> sp.csr_matrix:
    """S (M×N): one 1 per column — the hard-assignment splat (PAPER.md:107-112, :116 SSᵀ = Dm)."""
    N = vid.shape[0]
    return sp.csr_matrix((np.ones(N), (vid, np.arange(N))), shape=(M, N))


def blur_matrix(nbr: np.ndarray, dims: int = D) -> sp.csr_matrix:
    """B̄ = 2D·I + Σ_d (E_d⁺ + E_d⁻): sum of 1-D [1 2 1] blurs over the D grid dimensions
    (reading #4; D = 3 for a grayscale reference, reading #27)."""
    M = nbr.shape[0]
    rows, cols = np.nonzero(nbr >= 0)
    adj = sp.csr_matrix((np.ones(rows.size), (rows, nbr[rows, cols])), shape=(M, M))
    return (2 * dims * sp.identity(M, format="csr") + adj).tocsr()


def bistochastize(m: np.ndarray, Bbar: sp.csr_matrix, n_iters: int = 20):
    """Alg. 1 (Supp §1 Alg. bistoch), exactly ``n_iters`` iterations (reading #5):
        m ← S1;  n ← 1;  repeat: n ← sqrt((n ∘ m) / (B̄ n)).
    Returns (n, residual) with residual = max|n∘B̄n − m| / max m."""
    m = m.astype(np.float64)
    n = np.ones_like(m)
    for _ in range(n_iters):
        n = np.sqrt((n * m) / (Bbar @ n))
    residual = float(np.max(np.abs(n * (Bbar @ n) - m)) / np.max(m)) if m.size else 0.0
    return n, residual


# ----------------------------------------------------------------------------- system
@dataclass
class System:
    """Bilateral-space quadratic of one frame (PAPER.md:124-127 Eq. quad_min)."""

    A: sp.csr_matrix  # λ(Dm − Dn B̄ Dn) + diag(Sc), isolated-row rule (reading #6)
    b: np.ndarray  # [M][K]  b = S(c∘t)
    Sc: np.ndarray  # [M]     S c
    diagA: np.ndarray  # [M]
    live: np.ndarray  # bool [M]  not (isolated ∧ Sc = 0)   (reading #6)
    c0: np.ndarray  # [K]   ½ (c∘t)ᵀ t


def assemble(S: sp.csr_matrix, Bbar: sp.csr_matrix, m, n, nbr, t: np.ndarray, c: np.ndarray, lam: float) -> System:
    """A = λ(Dm − Dn B̄ Dn) + diag(S c),  b = S(c ∘ t),  c₀ = ½(c∘t)ᵀt.

    t: [K][N] targets, c: [N] confidence.  Reading #6: an isolated vertex (no
    neighbours) has a structurally zero smoothness row; its diagonal smoothness
    λ(m − 2D n²) is set to exactly 0 (rounding would otherwise leave ±ulp)."""
    m = m.astype(np.float64)
    Sc = S @ c
    b = np.stack([S @ (c * tk) for tk in t], axis=1)
    Dn = sp.diags(n)
    A_smooth = lam * (sp.diags(m) - Dn @ Bbar @ Dn)
    isolated = np.all(nbr < 0, axis=1)
    fix = np.where(isolated, -A_smooth.diagonal(), 0.0)
    A = (A_smooth + sp.diags(fix) + sp.diags(Sc)).tocsr()
    # diag(A) per PAPER.md:230: λ(diag Dm − diag Dn · B̄_diag · diag Dn) + S c
    bdiag = Bbar.diagonal()  # the constant 2D (reading #4)
    diagA = lam * (m - n * bdiag * n) + Sc
    diagA = np.where(isolated, Sc, diagA)
    live = ~(isolated & (Sc == 0))
    c0 = 0.5 * np.array([np.dot(c * tk, tk) for tk in t])
    return System(A=A, b=b, Sc=Sc, diagA=diagA, live=live, c0=c0)


def jacobi_minv(sysm: System) -> Callable[[np.ndarray], np.ndarray]:
    """M⁻¹_jacobi(y) = diag(A)⁻¹ y; 0 on dead vertices (reading #6)."""
    inv = np.where(sysm.live, 1.0 / np.where(sysm.live, sysm.diagA, 1.0), 0.0)
    return lambda r: inv * r


def flat_init(sysm: System) -> np.ndarray:
    """y_flat = S(c∘t) / S(c)  (PAPER.md:238-241 Eq. flat_init); 0 where S c = 0 (reading #9)."""
    den = sysm.Sc[:, None]
    return np.where(den > 0, sysm.b / np.where(den > 0, den, 1.0), 0.0)


# ----------------------------------------------------------------------------- pyramid
@dataclass
class Pyramid:
    """Bilateral-space pyramid (Supp §2; reading #8).

    levels[k] = vertex tuples of level k (level 0 = the grid's vertices);
    parents[k] maps level k → level k+1 (the splat matrix S_k as an index map)."""

    levels: List[np.ndarray]
    parents: List[np.ndarray]

    @property
    def K(self) -> int:
        return len(self.levels)

    def S(self, k: int) -> sp.csr_matrix:
        """Splat matrix S_k (M_{k+1} × M_k)."""
        return splat_matrix(self.parents[k], self.levels[k + 1].shape[0])


def build_pyramid(V: np.ndarray) -> Pyramid:
    """for k: V ← V/2; (S_k, V) ← simplified_bilateral_grid(V), until one vertex
    (PAPER.md:750-757).  Reading #8: integer coordinates halved with ⌊·/2⌋, the
    frame field is not halved, level k = 0 is the grid itself."""
    levels = [V.copy()]
    parents = []
    while levels[-1].shape[0] > 1:
        H = levels[-1].copy()
        H[:, 1:] //= 2
        Vn, parent = np.unique(H, axis=0, return_inverse=True)
        parents.append(parent.reshape(-1).astype(np.int64))
        levels.append(Vn)
    return Pyramid(levels=levels, parents=parents)


def P_lift(pyr: Pyramid, y: np.ndarray) -> List[np.ndarray]:
    """P(y) = [y, S_0 y, S_1 S_0 y, …]  (listed here base-first, index = level k)."""
    out = [y]
    for k in range(pyr.K - 1):
        out.append(pyr.S(k) @ out[-1])
    return out


def P_project(pyr: Pyramid, z: List[np.ndarray]) -> np.ndarray:
    """Pᵀ(z) = Σ_k S_0ᵀ S_1ᵀ … S_{k−1}ᵀ z_k, computed top-down."""
    acc = z[-1]
    for k in range(pyr.K - 2, -1, -1):
        acc = z[k] + pyr.S(k).T @ acc
    return acc


def z_weight(k: int, alpha: float, beta: float) -> float:
    """z_weight = 1 if k = 0 else α^−(β+k)."""
    return 1.0 if k == 0 else float(alpha) ** (-(beta + k))


def hier_minv(pyr: Pyramid, sysm: System, alpha=2.0, beta=5.0) -> Callable[[np.ndarray], np.ndarray]:
    """M⁻¹_hier(y) = Pᵀ( z_w ∘ P(1) ∘ P(y) / P(diag A) )  (PAPER.md:266-270 Eq. hier_precond),
    α = 2, β = 5.  Readings #6 and #10: dead vertices are masked out
    on input and output; quotients with a zero denominator are 0."""
    mask = sysm.live.astype(np.float64)
    P1 = P_lift(pyr, np.ones(pyr.levels[0].shape[0]))
    PdA = P_lift(pyr, sysm.diagA * mask)
    mu = [np.where(PdA[k] > 0, z_weight(k, alpha, beta) * P1[k] / np.where(PdA[k] > 0, PdA[k], 1.0), 0.0)
          for k in range(pyr.K)]

    def apply(r: np.ndarray) -> np.ndarray:
        Pr = P_lift(pyr, mask * r)
        return mask * P_project(pyr, [mu[k] * Pr[k] for k in range(pyr.K)])

    apply.mu = mu  # exposed for tests
    return apply


def hier_init(pyr: Pyramid, sysm: System, alpha=4.0, beta=0.0) -> np.ndarray:
    """y_hier = Pᵀ(z_w ∘ P(S(c∘t)) / P(1)) / Pᵀ(z_w ∘ P(S c) / P(1)),
    α = 4, β = 0; 0 where the denominator is 0 (reading #10)."""
    P1 = P_lift(pyr, np.ones(pyr.levels[0].shape[0]))
    w = [z_weight(k, alpha, beta) / P1[k] for k in range(pyr.K)]
    PSc = P_lift(pyr, sysm.Sc)
    den = P_project(pyr, [w[k] * PSc[k] for k in range(pyr.K)])
    out = np.zeros_like(sysm.b)
    for j in range(sysm.b.shape[1]):
        Pb = P_lift(pyr, sysm.b[:, j])
        num = P_project(pyr, [w[k] * Pb[k] for k in range(pyr.K)])
        out[:, j] = np.where(den > 0, num / np.where(den > 0, den, 1.0), 0.0)
    return out


# ----------------------------------------------------------------------------- PCG
@dataclass
class PCGResult:
    x: np.ndarray
    iterations: int
    relres: float  # recurrence ‖r‖/‖b‖ at exit (0 if ‖b‖ = 0 and r = 0)
    losses: List[float] = field(default_factory=list)


def pcg(A: Callable[[np.ndarray], np.ndarray], b: np.ndarray, x: np.ndarray,
        Minv: Callable[[np.ndarray], np.ndarray], n: int, tol: Optional[float] = None,
        track_loss: bool = False) -> PCGResult:
    """Alg. 2, PCG of Shewchuk B3, fp64, one right-hand side.

    FIXED (tol is None): exactly ``n`` iterations ("while i < n").
    TOL (reading #11): additionally stop when ‖r_i‖₂ ≤ tol·‖b‖₂, tested before every
    iteration including i = 0, with ``n`` as max_iters.  Breakdown guard: stop if
    ρ = 0 or dᵀq ≤ 0.  Reading #12: the paper's λ_new/λ_old are named ρ here."""
    x = x.astype(np.float64).copy()
    r = b - A(x)  # line 2
    d = Minv(r)  # line 3
    rho = float(r @ d)  # line 4
    bnorm = float(np.linalg.norm(b))
    losses = []
    i = 0
    while i < n:  # line 5
        if tol is not None and np.linalg.norm(r) <= tol * bnorm:
            break
        if rho == 0.0:
            break
        if track_loss:
            losses.append(0.5 * float(x @ A(x)) - float(b @ x))
        q = A(d)  # line 6
        dq = float(d @ q)
        if dq <= 0.0:
            break
        alpha = rho / dq  # line 7
        x = x + alpha * d  # line 8
        r = r - alpha * q  # line 9
        s = Minv(r)  # line 10
        rho_old = rho  # line 11
        rho = float(r @ s)  # line 12
        beta = rho / rho_old  # line 13
        d = s + beta * d  # line 14
        i += 1  # line 15
    if track_loss:
        losses.append(0.5 * float(x @ A(x)) - float(b @ x))
    relres = float(np.linalg.norm(r) / bnorm) if bnorm > 0 else float(np.linalg.norm(r))
    return PCGResult(x=x, iterations=i, relres=relres, losses=losses)


# ----------------------------------------------------------------------------- solve
@dataclass
class SolveOptions:
    precond: str = "jacobi"  # jacobi | hier
    init: str = "flat"  # flat | hier | zero
    mode: str = "tol"  # tol | fixed
    iters: int = 25  # FIXED count ("25 iterations of PCG")
    tol: float = 1e-6
    max_iters: int = 2000
    precond_alpha: float = 2.0
    precond_beta: float = 5.0
    init_alpha: float = 4.0
    init_beta: float = 0.0
    n_bistoch: int = 20  # reading #5


@dataclass
class FrameSolution:
    """Everything the oracle computes for one frame (vertex arrays in canonical order)."""

    V: np.ndarray
    m: np.ndarray
    nbr: np.ndarray  # frame-local indices
    n: np.ndarray
    bistoch_residual: float
    sys: System
    pyr: Optional[Pyramid]
    y0: np.ndarray  # [M][K]
    y: np.ndarray  # [M][K]
    x: np.ndarray  # [K][H*W]
    iterations: List[int]
    relres: List[float]
    Minv: Callable = field(repr=False, default=None)
    S: sp.csr_matrix = field(repr=False, default=None)
    vid: np.ndarray = field(repr=False, default=None)


def solve_frame(grid: Grid, f: int, t: np.ndarray, c: np.ndarray, lam: float,
                opts: SolveOptions, track_loss: bool = False) -> FrameSolution:
    """Bilateral solver for frame f: build system, init, PCG, slice
    (§2 "we construct a simplified bilateral grid …", Eq. solution :137-140).

    t: [K][H*W], c: [H*W] for this frame (row-major pixels)."""
    v0, v1 = int(grid.frame_start[f]), int(grid.frame_start[f + 1])
    HW = c.shape[0]
    vid = grid.vid[f * HW:(f + 1) * HW] - v0
    V = grid.V[v0:v1]
    m = grid.m[v0:v1]
    nbr = np.where(grid.nbr[v0:v1] >= 0, grid.nbr[v0:v1] - v0, -1)
    M = v1 - v0
    S = splat_matrix(vid, M)
    Bbar = blur_matrix(nbr, grid.dims)
    n, res = bistochastize(m, Bbar, opts.n_bistoch)
    sysm = assemble(S, Bbar, m, n, nbr, t, c, lam)
    pyr = build_pyramid(V) if (opts.precond == "hier" or opts.init == "hier") else None

    if opts.precond == "hier":
        Minv = hier_minv(pyr, sysm, opts.precond_alpha, opts.precond_beta)
    else:
        Minv = jacobi_minv(sysm)
    if opts.init == "hier":
        y0 = hier_init(pyr, sysm, opts.init_alpha, opts.init_beta)
    elif opts.init == "flat":
        y0 = flat_init(sysm)
    else:
        y0 = np.zeros_like(sysm.b)

    Aop = lambda v: sysm.A @ v  # noqa: E731
    K = t.shape[0]
    y = np.zeros_like(y0)
    iters, rel = [], []
    for k in range(K):
        if opts.mode == "fixed":
            r = pcg(Aop, sysm.b[:, k], y0[:, k], Minv, opts.iters, None, track_loss)
        else:
            r = pcg(Aop, sysm.b[:, k], y0[:, k], Minv, opts.max_iters, opts.tol, track_loss)
        y[:, k] = r.x
        iters.append(r.iterations)
        rel.append(r.relres)
    x = np.stack([S.T @ y[:, k] for k in range(K)])  # x̂ = Sᵀ ŷ
    return FrameSolution(V=V, m=m, nbr=nbr, n=n, bistoch_residual=res, sys=sysm, pyr=pyr,
                         y0=y0, y=y, x=x, iterations=iters, relres=rel, Minv=Minv, S=S, vid=vid)


def solve(rgb, t, c, sigma_xy, sigma_l, sigma_uv, lam, opts: SolveOptions, frames=None, dims: int = 5):
    """Batch entry: rgb [F][H][W][3], t [F][K][H][W], c [F][H][W] → (grid, [FrameSolution])."""
    F, H, W, _ = rgb.shape
    grid = build_grid(rgb, sigma_xy, sigma_l, sigma_uv, dims)
    sols = []
    for f in (range(F) if frames is None else frames):
        tf = t[f].reshape(t.shape[1], H * W).astype(np.float64)
        cf = c[f].reshape(H * W).astype(np.float64)
        sols.append(solve_frame(grid, f, tf, cf, lam, opts))
    return grid, sols


def solve_backward(sol: FrameSolution, g: np.ndarray, t: np.ndarray, c: np.ndarray,
                   opts: SolveOptions):
    """Backprop through the solver (§3, reading #14, #15):
        ∂f/∂b = A⁻¹(S ∂f/∂x̂)               solved with the forward's M⁻¹, from 0
        ∂f/∂diag(A) = −∂f/∂b ∘ ŷ
        ∂f/∂t = c ∘ Sᵀ ∂f/∂b
        ∂f/∂c = Sᵀ ∂f/∂diag(A) + (Sᵀ ∂f/∂b) ∘ t        (summed over channels)
    g, t: [K][H*W], c: [H*W].  Returns (dt [K][HW], dc [HW], d_b [M][K], iterations)."""
    S = sol.S
    K = g.shape[0]
    Aop = lambda v: sol.sys.A @ v  # noqa: E731
    dt = np.zeros_like(g, dtype=np.float64)
    dc = np.zeros(c.shape[0])
    db = np.zeros((S.shape[0], K))
    iters = []
    for k in range(K):
        u = S @ g[k]
        zero = np.zeros_like(u)
        if opts.mode == "fixed":
            r = pcg(Aop, u, zero, sol.Minv, opts.iters, None)
        else:
            r = pcg(Aop, u, zero, sol.Minv, opts.max_iters, opts.tol)
        db[:, k] = r.x
        iters.append(r.iterations)
        d_diagA = -r.x * sol.y[:, k]
        dt[k] = c * (S.T @ r.x)
        dc += S.T @ d_diagA + (S.T @ r.x) * t[k]
    return dt, dc, db, iters


# ----------------------------------------------------------------------------- robust (Supp. §3)
def gm_rho(e, sigma_gm: float):
    """Geman–McClure estimator ρ(e) = e² / (σ_gm² + e²)  (Supp. §3)."""
    e = np.asarray(e, dtype=np.float64)
    return e * e / (sigma_gm * sigma_gm + e * e)


def gm_weight(e, sigma_gm: float):
    """Its IRLS weight w(e) = 2σ_gm² / (σ_gm² + e²)²  (Alg. 3 line 5)."""
    e = np.asarray(e, dtype=np.float64)
    s2 = sigma_gm * sigma_gm
    return 2.0 * s2 / (s2 + e * e) ** 2


def smoothness(sol: FrameSolution) -> float:
    """λ/2 Σ_ij Ŵ_ij (x_i − x_j)² at x = Sᵀŷ, evaluated in bilateral space as ŷᵀ(A − diag(Sc))ŷ
    (reading #17: Eq.1(Sᵀy) = yᵀAy − 2bᵀy + (c∘t)ᵀt)."""
    y = sol.y[:, 0]
    return float(y @ (sol.sys.A @ y) - y @ (sol.sys.Sc * y))


@dataclass
class RobustSolution:
    sol: FrameSolution  # the last inner solve (its x is x̂)
    weights: np.ndarray  # c after the last update (Alg. 3 line 5), [H*W]
    losses: List[float]  # Eq. robust_loss after each inner solve
    mm_losses: List[float]  # λ/2 Σ Ŵ (x_i − x_j)² + 2 Σ ρ(e_i): what c ← w minimises exactly (reading #25)


def robust_solve_frame(grid: Grid, f: int, t: np.ndarray, c_init: np.ndarray, lam: float, opts: SolveOptions,
                       sigma_gm: float, n_irls: int) -> RobustSolution:
    """Alg. 3 "The Geman-McClure Robust Bilateral Solver", verbatim:
        c ← c_init;  repeat n times:  x̂ ← solve(t, c);  e ← x̂ − t;  c ← 2σ²/(σ² + e∘e)².
    Scalar targets only (t: [1][H*W]; reading #25).  The grid, n and the smoothness part of A
    are the same for every inner solve; only diag(S c) and b change."""
    assert t.shape[0] == 1 and n_irls >= 1 and sigma_gm > 0
    c = np.asarray(c_init, dtype=np.float64).copy()
    losses, mm = [], []
    sol = None
    for _ in range(n_irls):
        sol = solve_frame(grid, f, t, c, lam, opts)  # line 3
        e = sol.x[0] - t[0]  # line 4
        sm = smoothness(sol)
        losses.append(sm + float(gm_rho(e, sigma_gm).sum()))
        mm.append(sm + 2.0 * float(gm_rho(e, sigma_gm).sum()))
        c = gm_weight(e, sigma_gm)  # line 5
    return RobustSolution(sol=sol, weights=c, losses=losses, mm_losses=mm)


def robust_solve(rgb, t, c_init, sigma_xy, sigma_l, sigma_uv, lam, opts: SolveOptions, sigma_gm: float,
                 n_irls: int, frames=None):
    """Batch entry of Alg. 3: rgb [F][H][W][3], t [F][1][H][W], c_init [F][H][W]."""
    F, H, W, _ = rgb.shape
    grid = build_grid(rgb, sigma_xy, sigma_l, sigma_uv)
    out = []
    for f in (range(F) if frames is None else frames):
        tf = t[f].reshape(1, H * W).astype(np.float64)
        cf = c_init[f].reshape(H * W).astype(np.float64)
        out.append(robust_solve_frame(grid, f, tf, cf, lam, opts, sigma_gm, n_irls))
    return grid, out


# ----------------------------------------------------------------------------- low-rank RHS (Supp. §4)
@dataclass
class ReducedRHS:
    Q: np.ndarray  # [M][t] orthonormal columns  (Q̃ = Q'[:, :t])
    R: np.ndarray  # [t][K]                     (R̃ = (R' Pᵀ)[:t, :])
    t: int
    masses: np.ndarray  # m_i of the rows of R', non-increasing


def reduce_rhs(B: np.ndarray, eps: float) -> ReducedRHS:
    """Rank reduction of the right-hand sides B [M][K] (Supp. §4):
    B P = Q R (column-pivoted QR; scipy.linalg.qr as the library step), R' = rows of R Pᵀ
    sorted by non-increasing squared norm m_i with Q' = the columns of Q in the same order,
    t = the smallest count with Σ_{i<t} m_i ≥ (1 − ε) Σ_i m_i (reading #26: the displayed
    inequality is inverted relative to the prose), Q̃ = Q'[:, :t], R̃ = R'[:t, :]."""
    import scipy.linalg as sla
    assert 0.0 <= eps < 1.0
    M, K = B.shape
    Q, R, piv = sla.qr(B, mode="economic", pivoting=True)  # B[:, piv] = Q R
    RPt = np.zeros_like(R)
    RPt[:, piv] = R  # R Pᵀ: columns back in channel order
    m = np.sum(RPt * RPt, axis=1)
    order = np.argsort(-m, kind="stable")
    m = m[order]
    total = float(m.sum())
    if total == 0.0:
        return ReducedRHS(Q=np.zeros((M, 0)), R=np.zeros((0, K)), t=0, masses=m)
    cum = np.cumsum(m)
    t = int(np.searchsorted(cum, (1.0 - eps) * total - 1e-12 * total) + 1)
    t = min(t, K)
    return ReducedRHS(Q=Q[:, order[:t]], R=RPt[order[:t], :], t=t, masses=m)


def solve_frame_lowrank(grid: Grid, f: int, t: np.ndarray, c: np.ndarray, lam: float, opts: SolveOptions,
                        eps: float):
    """Y = (A⁻¹ Q̃) R̃ (Supp. §4): solve the t reduced systems A ỹ_i = Q̃_i (initialised and
    preconditioned as the full solve would be, with Q̃ in place of b) and expand by R̃;
    x̂ = Sᵀ Y.  Returns (x [K][H*W], Y [M][K], ReducedRHS)."""
    full = solve_frame(grid, f, t, c, lam, SolveOptions(**{**opts.__dict__, "mode": "fixed", "iters": 0}))
    red = reduce_rhs(full.sys.b, eps)
    sysr = System(A=full.sys.A, b=red.Q, Sc=full.sys.Sc, diagA=full.sys.diagA, live=full.sys.live,
                  c0=np.zeros(red.t))
    if opts.init == "hier":
        y0 = hier_init(full.pyr, sysr, opts.init_alpha, opts.init_beta)
    elif opts.init == "flat":
        y0 = flat_init(sysr)
    else:
        y0 = np.zeros_like(red.Q)
    Aop = lambda v: full.sys.A @ v  # noqa: E731
    Yr = np.zeros((full.sys.A.shape[0], red.t))
    for i in range(red.t):
        if opts.mode == "fixed":
            r = pcg(Aop, red.Q[:, i], y0[:, i], full.Minv, opts.iters, None)
        else:
            r = pcg(Aop, red.Q[:, i], y0[:, i], full.Minv, opts.max_iters, opts.tol)
        Yr[:, i] = r.x
    Y = Yr @ red.R
    x = np.stack([full.S.T @ Y[:, k] for k in range(Y.shape[1])])
    return x, Y, red


# ----------------------------------------------------------------------------- domain transform (post-filter)
def dt_sigmas(sigma_s: float, n_iters: int = 3) -> np.ndarray:
    """σ_i of pass i = 1..N of the recursive domain transform (reading #28, Gastal & Oliveira
    2011 as restated in SPEC.md:465-505):  σ_i = σ_s √3 2^(N−i) / √(4^N − 1)."""
    N = n_iters
    return np.array([sigma_s * np.sqrt(3.0) * 2.0 ** (N - i) / np.sqrt(4.0 ** N - 1.0) for i in range(1, N + 1)])


def dt_filter(signal: np.ndarray, rgb: np.ndarray, sigma_s: float, sigma_r: float, n_iters: int = 3) -> np.ndarray:
    """Edge-aware post-filter of the solver output: the recursive-filter (RF) domain transform of
    Gastal & Oliveira 2011, which the paper cites and applies to every result (PAPER.md:329,
    :333 σ'_xy, σ'_rgb; Supp. §3 "the recursive formulation of the domain transform"), restated
    from that publication (reading #28):
        d_x(p) = 1 + σ_s/σ_r Σ_c |I_c(p) − I_c(p − x̂)|   (L1 over RGB in [0, 255]; 1 at x = 0)
        pass i = 1..N:  σ_i = σ_s √3 2^(N−i) / √(4^N − 1),  a_i = exp(−√2 / σ_i),  w = a_i^d
          rows:    J[n] += w[n] (J[n−1] − J[n])  for n = 1 … W−1,  then
                   J[n] += w[n+1] (J[n+1] − J[n]) for n = W−2 … 0
          columns: the same with d_y.
    signal: [K][H][W], rgb: uint8 [H][W][3].  Returns float64 [K][H][W]."""
    F = np.array(signal, dtype=np.float64, copy=True)
    K, H, W = F.shape
    I = rgb.astype(np.float64)
    dx = np.zeros((H, W))
    dy = np.zeros((H, W))
    dx[:, 1:] = np.abs(np.diff(I, axis=1)).sum(axis=2)
    dy[1:, :] = np.abs(np.diff(I, axis=0)).sum(axis=2)
    Dx = 1.0 + sigma_s / sigma_r * dx
    Dy = 1.0 + sigma_s / sigma_r * dy
    for sig in dt_sigmas(sigma_s, n_iters):
        a = np.exp(-np.sqrt(2.0) / sig)
        V = a ** Dx
        for x in range(1, W):
            F[:, :, x] += V[:, x] * (F[:, :, x - 1] - F[:, :, x])
        for x in range(W - 2, -1, -1):
            F[:, :, x] += V[:, x + 1] * (F[:, :, x + 1] - F[:, :, x])
        V = a ** Dy
        for y in range(1, H):
            F[:, y, :] += V[y, :] * (F[:, y - 1, :] - F[:, y, :])
        for y in range(H - 2, -1, -1):
            F[:, y, :] += V[y + 1, :] * (F[:, y + 1, :] - F[:, y, :])
    return F


# ----------------------------------------------------------------------------- brute force helpers
def dense_W_hat(S: sp.csr_matrix, Bbar: sp.csr_matrix, m, n) -> np.ndarray:
    """Ŵ = Sᵀ Dm⁻¹ Dn B̄ Dn Dm⁻¹ S  (PAPER.md:114-117 Eq. equiv / :650-652 Eq. What). Tiny inputs only."""
    Sd = S.toarray()
    mid = np.diag(n / m) @ Bbar.toarray() @ np.diag(n / m)
    return Sd.T @ mid @ Sd


def pixel_loss(x: np.ndarray, W_hat: np.ndarray, c: np.ndarray, t: np.ndarray, lam: float) -> float:
    """Eq. pixel_loss: λ/2 Σ_ij Ŵ_ij (x_i − x_j)² + Σ_i c_i (x_i − t_i)²."""
    diff = x[:, None] - x[None, :]
    return 0.5 * lam * float(np.sum(W_hat * diff * diff)) + float(np.sum(c * (x - t) ** 2))


def zero_confidence_components(nbr: np.ndarray, Sc: np.ndarray) -> np.ndarray:
    """Reading #7: label vertices whose whole connected component (of the neighbour graph)
    has S c = 0 — there A is singular and the solution is defined only by the PCG path."""
    M = nbr.shape[0]
    rows, cols = np.nonzero(nbr >= 0)
    G = sp.csr_matrix((np.ones(rows.size), (rows, nbr[rows, cols])), shape=(M, M))
    ncomp, lab = sp.csgraph.connected_components(G, directed=False)
    has_conf = np.zeros(ncomp, bool)
    np.logical_or.at(has_conf, lab, Sc > 0)
    return ~has_conf[lab]


__all__ = [name for name in dir() if not name.startswith("_")]
