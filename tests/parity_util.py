"""Helpers shared by the GPU parity tests: run the CUDA path (through the C ABI) and the
fp64 oracle on the same seeded workload and compare them with north_star's tolerances."""
from __future__ import annotations

import numpy as np

import oracle as O

# north_star: max-abs ≤ 1e-3 × target range, RMS ≤ 1e-4 × target range (BASELINE.json)
MAX_TOL = 1e-3
RMS_TOL = 1e-4


def oracle_opts(w, **over):
    kw = dict(precond=w.precond, init=w.init, mode=w.mode, iters=w.iters, tol=w.tol, max_iters=w.max_iters,
              n_bistoch=w.n_bistoch)
    kw.update(over)
    return O.SolveOptions(**kw)


def gpu_opts(w, **over):
    kw = dict(precond=w.precond, init=w.init, mode=w.mode, iters=w.iters, tol=w.tol, max_iters=w.max_iters)
    kw.update(over)
    return kw


def target_range(t, c):
    """Reading #18: per channel, max − min of t over pixels with c > 0; 0 → max(1, max|t|)."""
    K = t.shape[0]
    out = np.zeros(K)
    for k in range(K):
        sel = t[k][c > 0]
        r = float(sel.max() - sel.min()) if sel.size else 0.0
        out[k] = r if r > 0 else max(1.0, float(np.abs(t[k]).max()))
    return out


def compare_x(x_gpu, x_ref, t, c, exclude=None):
    """x_*: [K][HW] one frame.  Returns (max_rel, rms_rel) over channels, relative to the range."""
    rng = target_range(t, c)
    worst_max, worst_rms = 0.0, 0.0
    for k in range(x_ref.shape[0]):
        d = np.abs(x_gpu[k].astype(np.float64) - x_ref[k])
        if exclude is not None:
            d = d[~exclude]
        worst_max = max(worst_max, float(d.max()) / rng[k])
        worst_rms = max(worst_rms, float(np.sqrt(np.mean(d * d))) / rng[k])
    return worst_max, worst_rms


def zero_conf_pixels(sol):
    """Pixels whose vertex lies in a zero-confidence component (reading #7) — parity unpinned there."""
    zc = O.zero_confidence_components(sol.nbr, sol.sys.Sc)
    return zc[sol.vid]


def pcg_fp32_storage(sol, iters, k=0):
    """Alg. 2 with the oracle's own operators (sol.sys.A, sol.Minv, sol.y0) and
    every PCG vector rounded to fp32 after it is formed (dots in fp64) — the arithmetic the CUDA
    path performs, used as the reference where the fixed-count iterate is unstable (reading #29).
    Returns the sliced per-pixel result of channel k."""
    f32 = lambda v: v.astype(np.float32).astype(np.float64)  # noqa: E731
    A, Minv = sol.sys.A, sol.Minv
    b = sol.sys.b[:, k]
    x = f32(sol.y0[:, k].astype(np.float64))
    r = f32(b - A @ x)
    d = f32(Minv(r))
    rho = float(r @ d)
    for _ in range(iters):
        if rho == 0.0:
            break
        q = f32(A @ d)
        dq = float(d @ q)
        if dq <= 0.0:
            break
        alpha = rho / dq
        x = f32(x + alpha * d)
        r = f32(r - alpha * q)
        s = f32(Minv(r))
        rho_old, rho = rho, float(r @ s)
        d = f32(s + (rho / rho_old) * d)
    return x[sol.vid]


def fixed_count_unstable(sol, iters, t, c, k=0):
    """Pixels where storing the PCG vectors in fp32 alone moves the fixed-count iterate of channel
    k by more than half the north_star bound (reading #29), and that fp32-storage reference."""
    x32 = pcg_fp32_storage(sol, iters, k)
    rng = target_range(t, c)[k]
    return np.abs(x32 - sol.x[k]) > 0.5 * MAX_TOL * rng, x32
