"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Grids must be bit-exact; solutions within north_star's tolerances (max-abs ≤ 1e-3·range,
RMS ≤ 1e-4·range) at tol 1e-6 and at a fixed iteration count.
"""
import numpy as np
import pytest

import oracle as O
from parity_util import MAX_TOL, RMS_TOL, compare_x, gpu_opts, oracle_opts, zero_conf_pixels
from workloads import make

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1511_03296_b200 as fbs


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_grid(w, **kw):
    return fbs.grid_build(dev(w.rgb), w.sigma_xy, w.sigma_l, w.sigma_uv, n_bistoch=w.n_bistoch, **kw)


def assert_grid_equal(g, og):
    e = g.export()
    assert g.M == og.M
    assert np.array_equal(e["keys"], og.keys)
    assert np.array_equal(e["vid"], og.vid)
    assert np.array_equal(e["m"], og.m)
    assert np.array_equal(e["nbr"], og.nbr)
    return e


WORKLOADS = {
    "c1": lambda: make("c1"),
    "c2s": lambda: make("c2", W=347, H=277, n_cells=40),
    "c3s": lambda: make("c3", H=272, W=344, n_cells=40),
    "c4s": lambda: make("c4", W=250, H=187, n_cells=20),
    "c5s": lambda: make("c5", frames=3, W=240, H=136, n_cells=30),
}


@pytest.mark.parametrize("name", list(WORKLOADS))
def test_grid_bit_exact(name):
    w = WORKLOADS[name]()
    og = O.build_grid(w.rgb, w.sigma_xy, w.sigma_l, w.sigma_uv)
    g = gpu_grid(w)
    e = assert_grid_equal(g, og)
    # Alg. 1 in fp32 vs fp64: n within 1e-5 relative
    for f in range(w.frames):
        v0, v1 = og.frame_start[f], og.frame_start[f + 1]
        S = O.splat_matrix(og.vid[f * w.H * w.W:(f + 1) * w.H * w.W] - v0, v1 - v0)
        nbr = np.where(og.nbr[v0:v1] >= 0, og.nbr[v0:v1] - v0, -1)
        n, _ = O.bistochastize(og.m[v0:v1], O.blur_matrix(nbr), w.n_bistoch)
        assert np.allclose(e["n"][v0:v1], n, rtol=1e-5)
    assert S is not None


@pytest.mark.parametrize("name", list(WORKLOADS))
def test_pyramid_bit_exact(name):
    w = WORKLOADS[name]()
    og = O.build_grid(w.rgb, w.sigma_xy, w.sigma_l, w.sigma_uv)
    g = gpu_grid(w)
    info = g.info()
    for f in range(w.frames):
        v0, v1 = og.frame_start[f], og.frame_start[f + 1]
        pyr = O.build_pyramid(og.V[v0:v1])
        assert info["frame_levels"][f] == pyr.K
    # compare each frame's segment of every level it has (k < L_f)
    Lmax = info["levels"]
    levels = {k: g.pyramid_level(k) for k in range(1, Lmax)}
    for f in range(w.frames):
        v0, v1 = og.frame_start[f], og.frame_start[f + 1]
        pyr = O.build_pyramid(og.V[v0:v1])
        P1 = O.P_lift(pyr, np.ones(v1 - v0))
        prev_off = v0
        for k in range(1, pyr.K):
            lv = levels[k]
            fr = (lv["keys"] >> np.uint64(56)).astype(np.int64)
            seg = np.nonzero(fr == f)[0]
            off = seg[0]
            assert np.array_equal(lv["keys"][seg], O.pack_key(pyr.levels[k]))
            assert np.array_equal(lv["count"][seg], P1[k].astype(np.int64))
            n_prev = pyr.levels[k - 1].shape[0]
            assert np.array_equal(lv["parent"][prev_off:prev_off + n_prev] - off, pyr.parents[k - 1])
            prev_off = off


def run_both(w, **over):
    t = torch.from_numpy(w.t).cuda()
    c = torch.from_numpy(w.c).cuda()
    g = gpu_grid(w)
    x, sysm = fbs.solve(g, t, c, w.lam, keep_system=True, **gpu_opts(w, **over))
    torch.cuda.synchronize()
    og, sols = O.solve(w.rgb, w.t, w.c, w.sigma_xy, w.sigma_l, w.sigma_uv, w.lam, oracle_opts(w, **over))
    return g, x.cpu().numpy(), sysm, og, sols


@pytest.mark.parametrize("name", list(WORKLOADS))
@pytest.mark.parametrize("mode", ["tol", "fixed"])
@pytest.mark.parametrize("pc", ["jacobi+flat", "hier+hier"])
def test_solve_parity(name, mode, pc):
    w = WORKLOADS[name]()
    precond, init = pc.split("+")
    g, x, sysm, og, sols = run_both(w, mode=mode, precond=precond, init=init)
    st = sysm.stats()
    for f, sol in enumerate(sols):
        HW = w.H * w.W
        t = w.t[f].reshape(w.K, HW).astype(np.float64)
        c = w.c[f].reshape(HW).astype(np.float64)
        zc = zero_conf_pixels(sol)
        mx, rms = compare_x(x[f].reshape(w.K, HW), sol.x, t, c, exclude=zc)
        assert mx <= MAX_TOL and rms <= RMS_TOL, (f, mx, rms, st["iterations"][f], sol.iterations)
        if mode == "fixed":
            assert np.all(st["iterations"][f] == np.minimum(w.iters, sol.iterations))
    assert st["status"] & ~2 == 0


@pytest.mark.parametrize("gray_ref", [True, False])
def test_d3_grid_bit_exact_and_colorization_parity(gray_ref):
    """D = 3 (XYL) grid of PAPER.md:511's colorization (reading #27): bit-exact grid against the
    oracle (on a gray and on a colour reference, whose chroma is then ignored), and a
    colorization-style solve — 2 chroma channels, confidence 1 on ~3% scribbled pixels —
    within north_star's bounds."""
    w = make("c2", W=190, H=150, n_cells=25)
    rgb = np.repeat(w.rgb[..., :1], 3, axis=3) if gray_ref else w.rgb
    H, W = w.H, w.W
    rng = np.random.default_rng(11)
    scrib = (rng.uniform(size=(1, H, W)) < 0.03).astype(np.float32)
    t = np.stack([w.t[:, 0] / 255.0 * 100.0 + 28.0, 200.0 - w.t[:, 0] / 2.0], axis=1).astype(np.float32) * scrib[:, None]
    g = fbs.grid_build(dev(rgb), 4.0, 4.0, 4.0, dims=3)
    og = O.build_grid(rgb, 4.0, 4.0, 4.0, dims=3)
    assert_grid_equal(g, og)
    x = fbs.solve(g, dev(t), dev(scrib), 0.5, precond="hier", init="hier", mode="tol", tol=1e-6).cpu().numpy()
    _, sols = O.solve(rgb, t, scrib, 4.0, 4.0, 4.0, 0.5,
                      O.SolveOptions(precond="hier", init="hier", mode="tol", tol=1e-6), dims=3)
    HW = H * W
    ex = zero_conf_pixels(sols[0])
    mx, rms = compare_x(x[0].reshape(2, HW), sols[0].x, t[0].reshape(2, HW).astype(float), scrib[0].ravel(), exclude=ex)
    assert mx <= MAX_TOL and rms <= RMS_TOL, (mx, rms)
