"""The whole step (grid build + FIXED-mode solve + release) is enqueue-only, so it can be captured
once into a CUDA graph and replayed on new inputs (§8(b) asynchrony; VERDICT r01 Missing #7).  The
replay must reproduce the eager call bit for bit, on the captured inputs and on new ones."""
import numpy as np
import pytest

from workloads import make

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1511_03296_b200 as fbs


@pytest.mark.parametrize("precond", ["hier", "jacobi"])
def test_step_graph_capture_and_replay(precond):
    init = "hier" if precond == "hier" else "flat"
    wa = make("c5", frames=3, W=240, H=136, n_cells=30)
    wb = make("c5", frames=3, W=240, H=136, n_cells=30, first_frame=3)
    dev = torch.device("cuda")
    rgb = torch.from_numpy(wa.rgb).to(dev)
    t = torch.from_numpy(wa.t).to(dev)
    c = torch.from_numpy(wa.c).to(dev)
    x = torch.empty_like(t)

    def step():
        g = fbs.grid_build(rgb, wa.sigma_xy, wa.sigma_l, wa.sigma_uv)
        fbs.solve(g, t, c, wa.lam, precond=precond, init=init, mode="fixed", iters=25, out=x)
        g.close()

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):  # warm-up outside the capture (one-time setup: streams, attributes)
            step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    eager_a = x.clone()
    graph = torch.cuda.CUDAGraph()
    l0 = fbs.launch_count()
    with torch.cuda.graph(graph):
        step()
    assert fbs.launch_count() > l0  # the library's kernels were captured
    x.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(x, eager_a)
    # new inputs into the captured buffers: the replay equals an eager call on them
    rgb.copy_(torch.from_numpy(wb.rgb))
    t.copy_(torch.from_numpy(wb.t))
    c.copy_(torch.from_numpy(wb.c))
    graph.replay()
    torch.cuda.synchronize()
    replay_b = x.clone()
    step()
    torch.cuda.synchronize()
    assert torch.equal(replay_b, x)
    assert not torch.equal(replay_b, eager_a)


@pytest.mark.parametrize("lowrank", [False, True])
def test_build_and_fixed_solve_only_enqueue(lowrank):
    """fbs_grid_build and a FIXED-mode fbs_solve (with or without the low-rank reduction) return
    while the stream is still busy: the calls never wait for the device (§8(b) asynchrony)."""
    import time
    w = make("c5", frames=2, W=160, H=96, n_cells=12)
    dev = torch.device("cuda")
    rgb = torch.from_numpy(w.rgb).to(dev)
    K = 4 if lowrank else 1
    t = torch.from_numpy(np.repeat(w.t, K, axis=1)).to(dev)
    c = torch.from_numpy(w.c).to(dev)
    kw = dict(precond="hier", init="hier", mode="fixed", iters=10, lowrank_eps=0.01 if lowrank else 0.0)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):  # warm-up (one-time set-up: streams, attributes, pools)
        g = fbs.grid_build(rgb, w.sigma_xy, w.sigma_l, w.sigma_uv)
        x_ref = fbs.solve(g, t, c, w.lam, **kw)
        g.close()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        torch.cuda._sleep(int(3e8))  # keep the stream busy for ~0.15 s
        h0 = time.perf_counter()
        g = fbs.grid_build(rgb, w.sigma_xy, w.sigma_l, w.sigma_uv)
        x = fbs.solve(g, t, c, w.lam, **kw)
        h1 = time.perf_counter()
        busy = not s.query()
    torch.cuda.synchronize()
    assert busy, "the stream finished before the calls returned: nothing was left to enqueue against"
    assert h1 - h0 < 0.05, f"the calls took {h1 - h0:.3f} s of host time: they waited for the device"
    assert torch.equal(x, x_ref)
    g.close()


@pytest.mark.parametrize("frames,precond", [(1, "hier"), (3, "hier"), (1, "jacobi")])
def test_tol_solve_graph_capture(frames, precond):
    """Inside a caller's CUDA-graph capture a TOL-mode solve becomes a device-side conditional while
    loop (no host polls), so the whole TOL step replays too; the replay equals the eager
    (host-polled) solve bit for bit, including the per-channel iteration counts."""
    init = "hier" if precond == "hier" else "flat"
    w = make("c5", frames=frames, W=200, H=120, n_cells=16)
    dev = torch.device("cuda")
    rgb, t, c = (torch.from_numpy(a).to(dev) for a in (w.rgb, w.t, w.c))
    kw = dict(precond=precond, init=init, mode="tol", tol=1e-6, max_iters=500)
    g0 = fbs.grid_build(rgb, w.sigma_xy, w.sigma_l, w.sigma_uv)
    x_eager, S0 = fbs.solve(g0, t, c, w.lam, keep_system=True, **kw)
    it_eager = S0.stats()["iterations"].copy()
    x = torch.empty_like(t)
    holder = {}

    def step():
        g = fbs.grid_build(rgb, w.sigma_xy, w.sigma_l, w.sigma_uv)
        _, S = fbs.solve(g, t, c, w.lam, keep_system=True, out=x, **kw)
        holder["S"], holder["g"] = S, g

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    # release the warm-up handles before capturing: destroying a handle enqueues frees on its own
    # (non-capturing) stream, which a global-mode capture in progress does not allow
    holder.clear()
    import gc
    gc.collect()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    x.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(x, x_eager)
    assert np.array_equal(holder["S"].stats()["iterations"], it_eager)
    assert np.all(it_eager > 1)
