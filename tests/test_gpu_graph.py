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
