"""GPU operator parity, backward parity, edge cases, determinism and error paths (C ABI)."""
import numpy as np
import pytest

import oracle as O
from parity_util import MAX_TOL, RMS_TOL, compare_x, gpu_opts, oracle_opts, target_range, zero_conf_pixels
from workloads import make
from workloads.synth import voronoi_reference

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1511_03296_b200 as fbs


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def small(K=3, seed=3, W=83, H=61, cells=9, frames=1):
    rng = np.random.default_rng(seed)
    rgbs = [voronoi_reference(rng, W, H, cells, "gradient", 3.0)[0] for _ in range(frames)]
    rgb = np.stack(rgbs)
    t = rng.uniform(0, 10, (frames, K, H, W)).astype(np.float32)
    c = rng.uniform(0.1, 1.0, (frames, H, W)).astype(np.float32)
    return rgb, t, c


def frame_oracle(rgb, t, c, lam, **kw):
    og = O.build_grid(rgb, 8.0, 4.0, 3.0)
    HW = rgb.shape[1] * rgb.shape[2]
    sol = O.solve_frame(og, 0, t[0].reshape(t.shape[1], HW).astype(float), c[0].ravel().astype(float), lam,
                        O.SolveOptions(**kw))
    return og, sol


# ----------------------------------------------------------------------------- operators
def test_splat_slice_blur():
    rgb, t, c = small(K=3, frames=2)
    g = fbs.grid_build(dev(rgb), 8.0, 4.0, 3.0)
    og = O.build_grid(rgb, 8.0, 4.0, 3.0)
    S = O.splat_matrix(og.vid, og.M)
    out = fbs.splat(g, dev(t)).cpu().numpy()
    N = rgb.shape[0] * rgb.shape[1] * rgb.shape[2]
    ref = np.stack([S @ t[:, k].reshape(N).astype(float) for k in range(3)], 1)
    assert np.allclose(out, ref, rtol=1e-6, atol=1e-5)
    ones = fbs.splat(g, torch.ones((2, 1, rgb.shape[1], rgb.shape[2]), device="cuda")).cpu().numpy()
    assert np.array_equal(ones[:, 0], og.m.astype(np.float32))  # S1 = m
    y = np.random.default_rng(1).normal(size=(og.M, 3)).astype(np.float32)
    x = fbs.slice_(g, dev(y)).cpu().numpy()
    assert np.array_equal(x.transpose(1, 0, 2, 3).reshape(3, N).T, y[og.vid])  # Sᵀy exact gather
    # adjointness ⟨S p, v⟩ = ⟨p, Sᵀ v⟩
    lhs = float(np.sum(out.astype(float) * y))
    rhs = float(np.sum(t.astype(float) * x.astype(float)))
    assert lhs == pytest.approx(rhs, rel=1e-5)
    v = np.random.default_rng(2).normal(size=og.M).astype(np.float32)
    bv = fbs.blur(g, dev(v)).cpu().numpy()
    assert np.allclose(bv, O.blur_matrix(og.nbr) @ v.astype(float), rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("precond", ["jacobi", "hier"])
def test_system_operators_and_exports(precond):
    rgb, t, c = small(K=2)
    lam = 50.0
    g = fbs.grid_build(dev(rgb), 8.0, 4.0, 3.0)
    x, s = fbs.solve(g, dev(t), dev(c), lam, keep_system=True, precond=precond, init="hier", mode="fixed", iters=5)
    og, sol = frame_oracle(rgb, t, c, lam, precond=precond, init="hier", mode="fixed", iters=5)
    e = s.export()
    assert np.allclose(e["sc"], sol.sys.Sc, rtol=1e-6)
    assert np.allclose(e["b"], sol.sys.b, rtol=1e-5, atol=1e-5)
    assert np.allclose(e["diagA"], sol.sys.diagA, rtol=1e-5)
    assert np.abs(e["y0"] - sol.y0).max() <= 1e-5 * np.abs(sol.y0).max()
    y = np.random.default_rng(4).normal(size=(og.M, 2)).astype(np.float32)
    Ay = s.apply_A(dev(y)).cpu().numpy()
    ref = sol.sys.A @ y.astype(float)
    assert np.abs(Ay - ref).max() <= 1e-5 * np.abs(sol.sys.diagA).max() * np.abs(y).max()
    My = s.apply_precond(dev(y)).cpu().numpy()
    refM = np.stack([sol.Minv(y[:, k].astype(float)) for k in range(2)], 1)
    assert np.abs(My - refM).max() <= 1e-5 * np.abs(refM).max()


# ----------------------------------------------------------------------------- backward
# Backward needs A SPD.  Config 3's zero-confidence components make A singular and
# S·g inconsistent there, so its backward is undefined in both implementations (reading #7).
BWD = {
    "c1": lambda: make("c1"),
    "c4s": lambda: make("c4", W=250, H=187, n_cells=20),
    "c2s": lambda: make("c2", W=347, H=277, n_cells=40),
}


@pytest.mark.parametrize("name", list(BWD))
@pytest.mark.parametrize("pc", ["jacobi+flat", "hier+hier"])
def test_backward_parity(name, pc):
    w = BWD[name]()
    precond, init = pc.split("+")
    over = dict(precond=precond, init=init, mode="tol", tol=1e-6)
    g = fbs.grid_build(dev(w.rgb), w.sigma_xy, w.sigma_l, w.sigma_uv)
    t, c = dev(w.t), dev(w.c)
    x, s = fbs.solve(g, t, c, w.lam, keep_system=True, **gpu_opts(w, **over))
    gr = w.g if w.g is not None else np.random.default_rng(1104).normal(size=w.t.shape).astype(np.float32)
    dt, dc = s.backward(dev(gr), t, c)
    dt, dc = dt.cpu().numpy(), dc.cpu().numpy()
    og, sols = O.solve(w.rgb, w.t, w.c, w.sigma_xy, w.sigma_l, w.sigma_uv, w.lam, oracle_opts(w, **over))
    sol = sols[0]
    HW = w.H * w.W
    odt, odc, odb, _ = O.solve_backward(sol, gr[0].reshape(w.K, HW).astype(float), w.t[0].reshape(w.K, HW).astype(float),
                                        w.c[0].ravel().astype(float), oracle_opts(w, **over))
    zc = zero_conf_pixels(sol)
    keep = ~zc
    rt = max(float(np.ptp(odt[:, keep])), 1e-30)
    d = np.abs(dt[0].reshape(w.K, HW) - odt)[:, keep]
    assert d.max() <= MAX_TOL * rt and np.sqrt(np.mean(d * d)) <= RMS_TOL * rt, (d.max() / rt)
    rc = max(float(np.ptp(odc[keep])), 1e-30)
    dcd = np.abs(dc[0].ravel() - odc)[keep]
    assert dcd.max() <= MAX_TOL * rc and np.sqrt(np.mean(dcd * dcd)) <= RMS_TOL * rc, (dcd.max() / rc)
    st = s.stats()
    assert np.all(st["bwd_iterations"] > 0)


def test_backward_scalar_example(worked):
    ex = worked["one_vertex"]
    rgb = np.broadcast_to(np.array(ex["rgb"], np.uint8), (1, 1, 2, 3)).copy()
    g = fbs.grid_build(dev(rgb), ex["sigma_xy"], ex["sigma_l"], ex["sigma_uv"])
    t = torch.tensor(ex["t"], dtype=torch.float32, device="cuda").reshape(1, 1, 1, 2)
    c = torch.tensor(ex["c"], dtype=torch.float32, device="cuda").reshape(1, 1, 2)
    x, s = fbs.solve(g, t, c, ex["lam"], keep_system=True, precond="jacobi", init="zero", mode="tol", tol=1e-7)
    assert np.allclose(x.cpu().numpy().ravel(), ex["x"], atol=1e-6)
    dt, dc = s.backward(torch.tensor(ex["g"], dtype=torch.float32, device="cuda").reshape(1, 1, 1, 2), t, c)
    assert np.allclose(dt.cpu().numpy().ravel(), ex["dt"], atol=1e-6)
    assert np.allclose(dc.cpu().numpy().ravel(), ex["dc"], atol=1e-6)


def test_two_vertex_example(worked):
    ex = worked["two_vertex_line"]
    rgb = np.broadcast_to(np.array(ex["rgb"], np.uint8), (1, 1, 2, 3)).copy()
    g = fbs.grid_build(dev(rgb), ex["sigma_xy"], ex["sigma_l"], ex["sigma_uv"])
    t = torch.tensor(ex["t"], dtype=torch.float32, device="cuda").reshape(1, 1, 1, 2)
    c = torch.tensor(ex["c"], dtype=torch.float32, device="cuda").reshape(1, 1, 2)
    x, s = fbs.solve(g, t, c, ex["lam"], keep_system=True, precond="hier", init="hier", mode="tol", tol=1e-7)
    assert np.allclose(x.cpu().numpy().ravel(), ex["y"], atol=1e-6)
    dt, dc = s.backward(torch.tensor(ex["g"], dtype=torch.float32, device="cuda").reshape(1, 1, 1, 2), t, c)
    assert np.allclose(dt.cpu().numpy().ravel(), ex["dt"], atol=1e-6)
    assert np.allclose(dc.cpu().numpy().ravel(), ex["dc"], atol=1e-6)


# ----------------------------------------------------------------------------- edge cases
@pytest.mark.parametrize("shape", [(1, 1), (1, 2), (2, 1), (1, 17), (13, 1), (9, 9), (33, 65)])
def test_tiny_and_ragged_shapes(shape):
    H, W = shape
    rng = np.random.default_rng(H * 100 + W)
    rgb = rng.integers(0, 256, (1, H, W, 3), dtype=np.uint8)
    t = rng.uniform(0, 1, (1, 1, H, W)).astype(np.float32)
    c = rng.uniform(0.1, 1, (1, H, W)).astype(np.float32)
    og = O.build_grid(rgb, 8.0, 4.0, 3.0)
    g = fbs.grid_build(dev(rgb), 8.0, 4.0, 3.0)
    e = g.export()
    assert np.array_equal(e["keys"], og.keys) and np.array_equal(e["vid"], og.vid)
    assert np.array_equal(e["nbr"], og.nbr) and np.array_equal(e["m"], og.m)
    x = fbs.solve(g, dev(t), dev(c), 10.0, precond="hier", init="hier", mode="tol", tol=1e-6).cpu().numpy()
    _, sol = frame_oracle(rgb, t, c, 10.0, precond="hier", init="hier", mode="tol", tol=1e-6)
    mx, rms = compare_x(x[0].reshape(1, -1), sol.x, t[0].reshape(1, -1).astype(float), c.ravel().astype(float))
    assert mx <= MAX_TOL and rms <= RMS_TOL


@pytest.mark.parametrize("sigmas", [(7.5, 4.0, 3.0), (1.0, 1.0, 1.0), (8.0, 16.0, 16.0), (2.5, 2.0, 5.5)])
def test_sigma_variants_bit_exact(sigmas):
    rgb, t, c = small(K=1, W=97, H=54)
    og = O.build_grid(rgb, *sigmas)
    g = fbs.grid_build(dev(rgb), *sigmas)
    e = g.export()
    assert np.array_equal(e["keys"], og.keys) and np.array_equal(e["vid"], og.vid)
    assert np.array_equal(e["nbr"], og.nbr) and np.array_equal(e["m"], og.m)


def test_noise_image_dense_grid():
    """Every pixel a distinct colour: M close to N, deep pyramid, dense coarse cells."""
    rng = np.random.default_rng(9)
    rgb = rng.integers(0, 256, (1, 64, 96, 3), dtype=np.uint8)
    og = O.build_grid(rgb, 8.0, 1.0, 1.0)
    g = fbs.grid_build(dev(rgb), 8.0, 1.0, 1.0)
    e = g.export()
    assert g.M == og.M and np.array_equal(e["keys"], og.keys) and np.array_equal(e["nbr"], og.nbr)


@pytest.mark.parametrize("sxy", [8.0, 5.0])
def test_noise_image_pyramid_bit_exact(sxy):
    """Dense coarse cells: level-1 coarse cells of up to 4·64 children (the largest register sort,
    E = 8) and level-2 ones of ~4·256 (noise keeps nearly every halved code distinct), which take
    the scratch path of k_pyr_sort.  Every level against the oracle's pyramid."""
    rng = np.random.default_rng(19)
    rgb = rng.integers(0, 256, (2, 80, 112, 3), dtype=np.uint8)
    og = O.build_grid(rgb, sxy, 1.0, 1.0)
    g = fbs.grid_build(dev(rgb), sxy, 1.0, 1.0)
    assert g.M == og.M
    info = g.info()
    levels = {k: g.pyramid_level(k) for k in range(1, info["levels"])}
    for f in range(rgb.shape[0]):
        v0, v1 = og.frame_start[f], og.frame_start[f + 1]
        pyr = O.build_pyramid(og.V[v0:v1])
        assert info["frame_levels"][f] == pyr.K
        P1 = O.P_lift(pyr, np.ones(v1 - v0))
        prev_off = v0
        for k in range(1, pyr.K):
            lv = levels[k]
            seg = np.nonzero((lv["keys"] >> np.uint64(56)).astype(np.int64) == f)[0]
            off = seg[0]
            assert np.array_equal(lv["keys"][seg], O.pack_key(pyr.levels[k]))
            assert np.array_equal(lv["count"][seg], P1[k].astype(np.int64))
            n_prev = pyr.levels[k - 1].shape[0]
            assert np.array_equal(lv["parent"][prev_off:prev_off + n_prev] - off, pyr.parents[k - 1])
            prev_off = off


def test_input_check_status_bits():
    """Negative confidence and non-finite inputs are flagged in the stats status word
    (FBS_ST_NEG_CONF = 4, FBS_ST_NONFINITE = 8), not silently solved."""
    rgb, t, c = small(K=1)
    g = fbs.grid_build(dev(rgb), 8.0, 4.0, 3.0)
    _, s = fbs.solve(g, dev(t), dev(c), 5.0, keep_system=True, mode="fixed", iters=3)
    assert s.stats()["status"] & 12 == 0
    c2 = c.copy()
    c2[0, 3, 4] = -0.5
    _, s = fbs.solve(g, dev(t), dev(c2), 5.0, keep_system=True, mode="fixed", iters=3)
    assert s.stats()["status"] & 4
    t2 = t.copy()
    t2[0, 0, 5, 6] = np.nan
    _, s = fbs.solve(g, dev(t2), dev(c), 5.0, keep_system=True, mode="fixed", iters=3)
    assert s.stats()["status"] & 8
    _, s = fbs.solve(g, dev(t), dev(c), 5.0, keep_system=True, mode="fixed", iters=3)
    gr = np.zeros_like(t)
    gr[0, 0, 1, 1] = np.inf
    s.backward(dev(gr), dev(t), dev(c))
    assert s.stats()["status"] & 8


def test_torch_caching_allocator():
    """Handles created after use_torch_allocator() take their buffers from PyTorch's caching
    allocator (visible in torch.cuda.memory_allocated) and return them on close; results are
    unchanged."""
    rgb, t, c = small(K=2)
    g0 = fbs.grid_build(dev(rgb), 8.0, 4.0, 3.0)
    x0 = fbs.solve(g0, dev(t), dev(c), 5.0, mode="fixed", iters=10)
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    fbs.use_torch_allocator(True)
    try:
        g = fbs.grid_build(dev(rgb), 8.0, 4.0, 3.0)
        torch.cuda.synchronize()
        held = torch.cuda.memory_allocated() - before
        assert held > 0
        x = fbs.solve(g, dev(t), dev(c), 5.0, mode="fixed", iters=10)
        assert torch.equal(x, x0)
        g.close()
        del x
        torch.cuda.synchronize()
    finally:
        fbs.use_torch_allocator(False)
    assert torch.cuda.memory_allocated() <= before + 4096


def test_allocator_callbacks_outlive_replacement():
    """A handle created under one registered allocator is destroyed after that allocator was
    replaced and then disabled: its callbacks must still be alive (fbs.py keeps every registered
    pair), so close() returns the buffers instead of jumping into a freed ctypes thunk."""
    rgb, t, c = small(K=1)
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    fbs.use_torch_allocator(True)
    try:
        g1 = fbs.grid_build(dev(rgb), 8.0, 4.0, 3.0)
        fbs.use_torch_allocator(True)  # a second registration replaces the first
        g2 = fbs.grid_build(dev(rgb), 8.0, 4.0, 3.0)
    finally:
        fbs.use_torch_allocator(False)
    import gc
    gc.collect()
    x = fbs.solve(g1, dev(t), dev(c), 5.0, mode="fixed", iters=5)
    g1.close()
    g2.close()
    del x
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated() <= before + 4096


def test_out_buffers_validated():
    """A caller-supplied out= of the wrong shape, dtype, layout or device is rejected before any
    kernel writes through it."""
    rgb, t, c = small(K=2)
    g = fbs.grid_build(dev(rgb), 8.0, 4.0, 3.0)
    T, Cc = dev(t), dev(c)
    good = torch.empty_like(T)
    fbs.solve(g, T, Cc, 5.0, mode="fixed", iters=3, out=good)
    for bad, exc in ((torch.empty(T.shape[0], 1, *T.shape[2:], device="cuda"), ValueError),
                     (torch.empty_like(T, dtype=torch.float64), TypeError),
                     (torch.empty(T.shape[::-1], device="cuda").permute(3, 2, 1, 0), ValueError),
                     (torch.empty_like(T, device="cpu"), TypeError)):
        with pytest.raises(exc):
            fbs.solve(g, T, Cc, 5.0, mode="fixed", iters=3, out=bad)
        with pytest.raises(exc):
            fbs.dt_filter(dev(rgb), T, 8.0, 8.0, out=bad)
    T1 = T[:, :1].contiguous()
    with pytest.raises(ValueError):
        fbs.solve_robust(g, T1, Cc, 5.0, 10.0, 1, mode="fixed", iters=3, out=torch.empty_like(T))


def test_zero_confidence_and_constant_target():
    rgb, t, c = small(K=2)
    g = fbs.grid_build(dev(rgb), 8.0, 4.0, 3.0)
    x, s = fbs.solve(g, dev(t), dev(np.zeros_like(c)), 5.0, keep_system=True, precond="hier", init="hier",
                     mode="tol", tol=1e-6)
    assert torch.all(x == 0) and np.all(s.stats()["iterations"] == 0)  # b = 0 → converged at i = 0
    x = fbs.solve(g, dev(np.full_like(t, 7.5)), dev(c), 5.0, precond="jacobi", init="flat", mode="tol", tol=1e-6)
    assert torch.allclose(x, torch.full_like(x, 7.5), atol=1e-4)


def test_identical_frames_identical_outputs_and_determinism():
    rgb, t, c = small(K=1, frames=1)
    rgb2, t2, c2 = np.concatenate([rgb, rgb]), np.concatenate([t, t]), np.concatenate([c, c])
    g = fbs.grid_build(dev(rgb2), 8.0, 4.0, 3.0)
    x1 = fbs.solve(g, dev(t2), dev(c2), 20.0, precond="hier", init="hier", mode="fixed", iters=25)
    x2 = fbs.solve(g, dev(t2), dev(c2), 20.0, precond="hier", init="hier", mode="fixed", iters=25)
    assert torch.equal(x1, x2)  # bitwise reproducible (fixed-order reductions)
    assert torch.equal(x1[0], x1[1])  # frames are independent systems
    g1 = fbs.grid_build(dev(rgb), 8.0, 4.0, 3.0)
    x3 = fbs.solve(g1, dev(t), dev(c), 20.0, precond="hier", init="hier", mode="fixed", iters=25)
    assert torch.equal(x3[0], x1[0])  # batch composition does not change a frame's result


def test_many_channels_k64():
    rgb, t, c = small(K=64, W=40, H=32)
    g = fbs.grid_build(dev(rgb), 8.0, 4.0, 3.0)
    x = fbs.solve(g, dev(t), dev(c), 5.0, precond="jacobi", init="flat", mode="fixed", iters=10).cpu().numpy()
    _, sol = frame_oracle(rgb, t, c, 5.0, precond="jacobi", init="flat", mode="fixed", iters=10)
    mx, rms = compare_x(x[0].reshape(64, -1), sol.x, t[0].reshape(64, -1).astype(float), c.ravel().astype(float))
    assert mx <= MAX_TOL and rms <= RMS_TOL


@pytest.mark.parametrize("pc", ["hier+hier", "jacobi+flat"])
def test_channel_joint_spmv(monkeypatch, pc):
    """The channel-joint SpMV (FBS_SPMV_K=joint: one neighbour-structure read per vertex for all K
    channels, north_star) gives the oracle's solution like the default channel-split kernel."""
    precond, init = pc.split("+")
    rgb, t, c = small(K=5, frames=2, W=50, H=37, cells=6)
    og = O.build_grid(rgb, 8.0, 4.0, 3.0)
    g = fbs.grid_build(dev(rgb), 8.0, 4.0, 3.0)
    monkeypatch.setenv("FBS_SPMV_K", "joint")
    l0 = fbs.launch_count()
    fbs.profile_reset()
    fbs.profile_enable(True)
    x = fbs.solve(g, dev(t), dev(c), 7.0, precond=precond, init=init, mode="fixed", iters=20).cpu().numpy()
    fbs.profile_enable(False)
    assert "k_spmv_kjoint" in fbs.profile_report() and fbs.launch_count() > l0
    for f in range(2):
        sol = O.solve_frame(og, f, t[f].reshape(5, -1).astype(float), c[f].ravel().astype(float), 7.0,
                            O.SolveOptions(precond=precond, init=init, mode="fixed", iters=20))
        mx, rms = compare_x(x[f].reshape(5, -1), sol.x, t[f].reshape(5, -1).astype(float), c[f].ravel().astype(float))
        assert mx <= MAX_TOL and rms <= RMS_TOL, (f, mx, rms)


def test_many_frames():
    rgb, t, c = small(K=1, frames=17, W=24, H=16, cells=4)
    og = O.build_grid(rgb, 8.0, 4.0, 3.0)
    g = fbs.grid_build(dev(rgb), 8.0, 4.0, 3.0)
    e = g.export()
    assert np.array_equal(e["keys"], og.keys) and np.array_equal(e["vid"], og.vid)
    x = fbs.solve(g, dev(t), dev(c), 5.0, precond="hier", init="hier", mode="tol", tol=1e-6).cpu().numpy()
    for f in range(17):
        sol = O.solve_frame(og, f, t[f].reshape(1, -1).astype(float), c[f].ravel().astype(float), 5.0,
                            O.SolveOptions(precond="hier", init="hier", mode="tol", tol=1e-6))
        mx, rms = compare_x(x[f].reshape(1, -1), sol.x, t[f].reshape(1, -1).astype(float), c[f].ravel().astype(float))
        assert mx <= MAX_TOL and rms <= RMS_TOL


@pytest.mark.parametrize("mode", ["fixed", "tol"])
@pytest.mark.parametrize("pc", ["hier+hier", "jacobi+flat"])
def test_frame_groups_times_channel_split(mode, pc):
    """Several frames (frame groups on side streams) × several channels (channel-split kernels,
    per-(frame, channel) counters and scalars), against per-frame oracle solves."""
    precond, init = pc.split("+")
    rgb, t, c = small(K=3, frames=5, W=70, H=45, cells=7)
    og = O.build_grid(rgb, 8.0, 4.0, 3.0)
    g = fbs.grid_build(dev(rgb), 8.0, 4.0, 3.0)
    x, S = fbs.solve(g, dev(t), dev(c), 7.0, keep_system=True, precond=precond, init=init, mode=mode, iters=25,
                     tol=1e-6)
    x = x.cpu().numpy()
    it = S.stats()["iterations"]
    for f in range(5):
        sol = O.solve_frame(og, f, t[f].reshape(3, -1).astype(float), c[f].ravel().astype(float), 7.0,
                            O.SolveOptions(precond=precond, init=init, mode=mode, iters=25, tol=1e-6))
        mx, rms = compare_x(x[f].reshape(3, -1), sol.x, t[f].reshape(3, -1).astype(float), c[f].ravel().astype(float))
        assert mx <= MAX_TOL and rms <= RMS_TOL, (f, mx, rms)
        if mode == "fixed":
            assert np.all(it[f] == np.minimum(25, sol.iterations))


def test_error_paths():
    rgb, t, c = small(K=1)
    with pytest.raises(fbs.FbsError) as e:
        fbs.grid_build(dev(rgb), 9.0, 4.0, 3.0)  # σxy > 8: cells would exceed 64 px
    assert e.value.code == 1
    with pytest.raises(fbs.FbsError):
        fbs.grid_build(dev(rgb), 8.0, 0.5, 3.0)  # σl < 1
    g = fbs.grid_build(dev(rgb), 8.0, 4.0, 3.0)
    with pytest.raises(fbs.FbsError):
        fbs.solve(g, dev(t), dev(c), 0.0)  # λ must be > 0
    with pytest.raises(fbs.FbsError):
        fbs.solve(g, dev(np.zeros((1, 65, rgb.shape[1], rgb.shape[2]), np.float32)), dev(c), 1.0)  # K > 64
    g2 = fbs.grid_build(dev(rgb), 8.0, 4.0, 3.0, build_pyramid=False)
    with pytest.raises(fbs.FbsError):
        fbs.solve(g2, dev(t), dev(c), 1.0, precond="hier")
    fbs.solve(g2, dev(t), dev(c), 1.0, precond="jacobi", init="flat")  # fine without a pyramid


def test_frame_field_limits():
    """256 frames (the 8-bit frame field of the key, reading #3) build bit-exactly, including
    frame 255, and solve frame-independently; 257 frames are rejected."""
    rng = np.random.default_rng(256)
    rgb = rng.integers(0, 256, (256, 9, 10, 3), dtype=np.uint8)
    og = O.build_grid(rgb, 4.0, 8.0, 8.0)
    g = fbs.grid_build(dev(rgb), 4.0, 8.0, 8.0)
    e = g.export()
    assert g.M == og.M and np.array_equal(e["keys"], og.keys) and np.array_equal(e["nbr"], og.nbr)
    assert int(e["keys"][-1] >> np.uint64(56)) == 255
    t = rng.uniform(0, 1, (256, 1, 9, 10)).astype(np.float32)
    c = np.ones((256, 9, 10), np.float32)
    x = fbs.solve(g, dev(t), dev(c), 2.0, precond="hier", init="hier", mode="fixed", iters=10).cpu().numpy()
    for f in (0, 128, 255):
        sol = O.solve_frame(og, f, t[f].reshape(1, -1).astype(float), c[f].ravel().astype(float), 2.0,
                            O.SolveOptions(precond="hier", init="hier", mode="fixed", iters=10))
        mx, rms = compare_x(x[f].reshape(1, -1), sol.x, t[f].reshape(1, -1).astype(float), c[f].ravel().astype(float))
        assert mx <= MAX_TOL and rms <= RMS_TOL, (f, mx, rms)
    with pytest.raises(fbs.FbsError):
        fbs.grid_build(dev(np.zeros((257, 4, 4, 3), np.uint8)), 4.0, 8.0, 8.0)


def test_empty_inputs_rejected():
    """Empty batches, planes and channel counts are argument errors (FBS_EINVAL), not crashes."""
    with pytest.raises(fbs.FbsError) as e:
        fbs.grid_build(dev(np.zeros((0, 8, 8, 3), np.uint8)), 8.0, 4.0, 3.0)
    assert e.value.code == 1
    for shape in [(1, 0, 8, 3), (1, 8, 0, 3)]:
        with pytest.raises(fbs.FbsError):
            fbs.grid_build(dev(np.zeros(shape, np.uint8)), 8.0, 4.0, 3.0)
    rgb, t, c = small(K=1)
    g = fbs.grid_build(dev(rgb), 8.0, 4.0, 3.0)
    with pytest.raises(fbs.FbsError):
        fbs.solve(g, dev(np.zeros((1, 0, rgb.shape[1], rgb.shape[2]), np.float32)), dev(c), 1.0)  # K = 0


@pytest.mark.parametrize("value", [0, 128, 255])
def test_constant_image(value):
    """A flat reference: one vertex per σxy cell (plus none in l, u, v), grid bit-exact, and the
    solve equals the oracle's (the degenerate case where only x/y neighbours exist)."""
    rgb = np.full((2, 37, 53, 3), value, np.uint8)
    og = O.build_grid(rgb, 8.0, 4.0, 3.0)
    g = fbs.grid_build(dev(rgb), 8.0, 4.0, 3.0)
    e = g.export()
    assert g.M == og.M == 2 * 5 * 7 and np.array_equal(e["keys"], og.keys) and np.array_equal(e["nbr"], og.nbr)
    rng = np.random.default_rng(value)
    t = rng.uniform(0, 1, (2, 1, 37, 53)).astype(np.float32)
    c = rng.uniform(0.1, 1, (2, 37, 53)).astype(np.float32)
    x = fbs.solve(g, dev(t), dev(c), 3.0, precond="hier", init="hier", mode="tol", tol=1e-6).cpu().numpy()
    for f in range(2):
        sol = O.solve_frame(og, f, t[f].reshape(1, -1).astype(float), c[f].ravel().astype(float), 3.0,
                            O.SolveOptions(precond="hier", init="hier", mode="tol", tol=1e-6))
        mx, rms = compare_x(x[f].reshape(1, -1), sol.x, t[f].reshape(1, -1).astype(float), c[f].ravel().astype(float))
        assert mx <= MAX_TOL and rms <= RMS_TOL, (f, mx, rms)


def test_tol_device_graph_loop(monkeypatch):
    """FBS_TOL_GRAPH=1: the TOL loop as a CUDA graph with a conditional while node (no host polls)
    gives the same iteration counts and results as the host-polled loop."""
    rgb, t, c = small(K=2, frames=1)
    g = fbs.grid_build(dev(rgb), 8.0, 4.0, 3.0)
    opts = dict(precond="hier", init="hier", mode="tol", tol=1e-6)
    x0, s0 = fbs.solve(g, dev(t), dev(c), 6.0, keep_system=True, **opts)
    monkeypatch.setenv("FBS_TOL_GRAPH", "1")
    x1, s1 = fbs.solve(g, dev(t), dev(c), 6.0, keep_system=True, **opts)
    monkeypatch.delenv("FBS_TOL_GRAPH")
    assert np.array_equal(s0.stats()["iterations"], s1.stats()["iterations"])
    assert torch.equal(x0, x1)


def test_launch_counter_and_profile():
    rgb, t, c = small(K=1)
    n0 = fbs.launch_count()
    fbs.profile_reset()
    fbs.profile_enable(True)
    g = fbs.grid_build(dev(rgb), 8.0, 4.0, 3.0)
    fbs.solve(g, dev(t), dev(c), 1.0, precond="jacobi", init="flat", mode="fixed", iters=3)
    torch.cuda.synchronize()
    fbs.profile_enable(False)
    rep = fbs.profile_report()
    assert fbs.launch_count() > n0
    assert rep["k_grid_sort"][0] == 1
    if rgb.shape[1] * rgb.shape[2] <= 98304:  # a small-frame Jacobi solve: one launch
        assert rep.get("k_pcg_small", (0,))[0] + rep.get("k_pcg_cluster", (0,))[0] == 1 and "k_spmv2" not in rep
    else:
        assert rep["k_spmv2"][0] == 3 and rep["k_direction2"][0] == 3
    assert sum(v[0] for v in rep.values()) == fbs.launch_count() - n0


def test_large_frame_tile_base_path(monkeypatch):
    """Frames with more level-1 scan tiles than the coarse kernel scans in shared memory take their
    tile bases from the lift's last block (k_tree_lift settle); forcing every frame onto that path
    (FBS_COARSE_TILES=0) gives bit-identical results, multi-frame and multi-channel."""
    rgb, t, c = small(K=3, frames=3, W=120, H=90, cells=9)
    g = fbs.grid_build(dev(rgb), 8.0, 4.0, 3.0)
    kw = dict(precond="hier", init="hier", mode="fixed", iters=12)
    x0 = fbs.solve(g, dev(t), dev(c), 6.0, **kw)
    monkeypatch.setenv("FBS_COARSE_TILES", "0")
    x1 = fbs.solve(g, dev(t), dev(c), 6.0, **kw)
    x2 = fbs.solve(g, dev(t[:, :1]), dev(c), 6.0, **kw)
    monkeypatch.delenv("FBS_COARSE_TILES")
    x3 = fbs.solve(g, dev(t[:, :1]), dev(c), 6.0, **kw)
    assert torch.equal(x0, x1) and torch.equal(x2, x3)
