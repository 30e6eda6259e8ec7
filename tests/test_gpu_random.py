"""Seeded random cases: grid, pyramid and solve parity on shapes, σ's and images none of the
BASELINE workloads use (odd sizes, partial edge cells, several frames of different content,
σxy from 1 to 8 and σl, σuv up to 32, noise mixed with flat regions).

The grid and pyramid must be bit-exact (north_star); the solve within north_star's bounds
(max-abs ≤ 1e-3·range, RMS ≤ 1e-4·range) against the fp64 oracle run to the same tolerance.
"""
import numpy as np
import pytest

import oracle as O
from parity_util import MAX_TOL, RMS_TOL, compare_x, zero_conf_pixels

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1511_03296_b200 as fbs


def case(seed):
    """A seeded random problem: frames of flat blocks, gradients and noise (the structure mix of the
    paper's references), a piecewise-smooth target of 1 or 3 channels and a confidence with exact
    zeros."""
    rng = np.random.default_rng(seed)
    F = int(rng.integers(1, 4))
    H = int(rng.integers(5, 97))
    W = int(rng.integers(5, 131))
    sxy = float(rng.choice([1.0, 2.0, 3.5, 5.0, 7.25, 8.0]))
    sl = float(rng.choice([1.0, 2.5, 4.0, 8.0, 32.0]))
    suv = float(rng.choice([1.0, 3.0, 4.5, 16.0]))
    K = int(rng.choice([1, 1, 3]))
    yy, xx = np.mgrid[0:H, 0:W]
    rgb = np.empty((F, H, W, 3), np.uint8)
    t = np.empty((F, K, H, W), np.float32)
    c = np.empty((F, H, W), np.float32)
    for f in range(F):
        blocks = rng.integers(0, 256, size=(4, 4, 3))
        base = blocks[(yy * 4) // H, (xx * 4) // W].astype(np.float64)
        base += rng.uniform(-1, 1, 3) * xx[..., None] + rng.uniform(-1, 1, 3) * yy[..., None]
        base += rng.normal(0, float(rng.choice([0.0, 3.0, 25.0])), base.shape)
        rgb[f] = np.clip(np.rint(base), 0, 255).astype(np.uint8)
        for k in range(K):
            t[f, k] = (rng.uniform(0, 10) + rng.uniform(-0.1, 0.1) * xx + rng.uniform(-0.1, 0.1) * yy
                       + rng.normal(0, 0.5, (H, W))).astype(np.float32)
        cf = rng.uniform(0.05, 1.0, (H, W))
        cf[rng.uniform(size=(H, W)) < 0.2] = 0.0
        c[f] = cf.astype(np.float32)
    return rgb, t, c, (sxy, sl, suv), float(rng.choice([1.0, 16.0, 128.0]))


SEEDS = list(range(101, 113))


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("seed", SEEDS)
def test_random_grid_and_pyramid_bit_exact(seed):
    rgb, _, _, sig, _ = case(seed)
    F, H, W = rgb.shape[:3]
    g = fbs.grid_build(dev(rgb), *sig)
    og = O.build_grid(rgb, *sig)
    e = g.export()
    assert g.M == og.M
    for k in ("keys", "vid", "m", "nbr"):
        assert np.array_equal(e[k], getattr(og, k)), k
    info = g.info()
    levels = {k: g.pyramid_level(k) for k in range(1, info["levels"])}
    for f in range(F):
        v0, v1 = og.frame_start[f], og.frame_start[f + 1]
        pyr = O.build_pyramid(og.V[v0:v1])
        assert info["frame_levels"][f] == pyr.K
        P1 = O.P_lift(pyr, np.ones(v1 - v0))
        for k in range(1, pyr.K):
            lv = levels[k]
            seg = np.nonzero((lv["keys"] >> np.uint64(56)).astype(np.int64) == f)[0]
            assert np.array_equal(lv["keys"][seg], O.pack_key(pyr.levels[k]))
            assert np.array_equal(lv["count"][seg], P1[k].astype(np.int64))
    g.close()


@pytest.mark.parametrize("seed", SEEDS)
@pytest.mark.parametrize("pc", ["hier+hier", "jacobi+flat"])
def test_random_solve_parity(seed, pc):
    rgb, t, c, sig, lam = case(seed)
    F, H, W = rgb.shape[:3]
    K = t.shape[1]
    precond, init = pc.split("+")
    g = fbs.grid_build(dev(rgb), *sig)
    x = fbs.solve(g, dev(t), dev(c), lam, precond=precond, init=init, mode="tol", tol=1e-6,
                  max_iters=5000).cpu().numpy()
    _, sols = O.solve(rgb, t, c, *sig, lam, O.SolveOptions(precond=precond, init=init, mode="tol", tol=1e-6,
                                                           max_iters=5000))
    HW = H * W
    for f, sol in enumerate(sols):
        mx, rms = compare_x(x[f].reshape(K, HW), sol.x, t[f].reshape(K, HW).astype(np.float64),
                            c[f].reshape(HW).astype(np.float64), exclude=zero_conf_pixels(sol))
        assert mx <= MAX_TOL and rms <= RMS_TOL, (seed, f, mx, rms)
    g.close()


@pytest.mark.parametrize("seed", SEEDS[:6])
@pytest.mark.parametrize("pc", ["hier+hier", "jacobi+flat"])
def test_random_backward_parity(seed, pc):
    """fbs_solve_backward against the oracle's; confidences kept > 0 so that
    S g is consistent on every component (reading #7: otherwise the backward is undefined)."""
    rgb, t, c, sig, lam = case(seed)
    c = np.maximum(c, 0.05).astype(np.float32)
    F, H, W = rgb.shape[:3]
    K = t.shape[1]
    HW = H * W
    precond, init = pc.split("+")
    opts = dict(precond=precond, init=init, mode="tol", tol=1e-6, max_iters=5000)
    gr = np.random.default_rng(seed + 7).normal(size=t.shape).astype(np.float32)
    g = fbs.grid_build(dev(rgb), *sig)
    td, cd = dev(t), dev(c)
    _, S = fbs.solve(g, td, cd, lam, keep_system=True, **opts)
    dt, dc = S.backward(dev(gr), td, cd)
    dt, dc = dt.cpu().numpy(), dc.cpu().numpy()
    _, sols = O.solve(rgb, t, c, *sig, lam, O.SolveOptions(**opts))
    for f, sol in enumerate(sols):
        odt, odc, _, _ = O.solve_backward(sol, gr[f].reshape(K, HW).astype(float), t[f].reshape(K, HW).astype(float),
                                          c[f].ravel().astype(float), O.SolveOptions(**opts))
        rt = max(float(np.ptp(odt)), 1e-30)
        d = np.abs(dt[f].reshape(K, HW) - odt)
        assert d.max() <= MAX_TOL * rt and np.sqrt(np.mean(d * d)) <= RMS_TOL * rt, (seed, f, d.max() / rt)
        # ∂c = Sᵀ(−d∘ŷ) + (Sᵀd)∘t: where ŷ = t exactly (a vertex of one pixel, flat init) the two
        # terms cancel and the oracle's ∂c is 0 — its scale is then that of the terms, |(Sᵀd)∘t|
        term = np.abs(odt / c[f].ravel() * t[f].reshape(K, HW)).sum(axis=0)
        rc = max(float(np.ptp(odc)), float(term.max()), 1e-30)
        dd = np.abs(dc[f].ravel() - odc)
        assert dd.max() <= MAX_TOL * rc and np.sqrt(np.mean(dd * dd)) <= RMS_TOL * rc, (seed, f, dd.max() / rc)
    S.close()
    g.close()
