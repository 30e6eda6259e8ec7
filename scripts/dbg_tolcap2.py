"""DEBUG: the TOL capture test's sequence, with the capture status checked after each call."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1511_03296_b200 as fbs
from workloads import make

w = make("c5", frames=1, W=200, H=120, n_cells=16)
dev = torch.device("cuda")
rgb, t, c = (torch.from_numpy(a).to(dev) for a in (w.rgb, w.t, w.c))
kw = dict(precond="hier", init="hier", mode="tol", tol=1e-6, max_iters=500)
g0 = fbs.grid_build(rgb, w.sigma_xy, w.sigma_l, w.sigma_uv)
x_eager, S0 = fbs.solve(g0, t, c, w.lam, keep_system=True, **kw)
print("eager iters", S0.stats()["iterations"], flush=True)
x = torch.empty_like(t)
holder = {}
variant = sys.argv[1] if len(sys.argv) > 1 else "full"


def step():
    g = fbs.grid_build(rgb, w.sigma_xy, w.sigma_l, w.sigma_uv)
    _, S = fbs.solve(g, t, c, w.lam, keep_system=True, out=x, **kw)
    holder["S"], holder["g"] = S, g


if variant != "nowarm":
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    print("warm ok", flush=True)
    if variant == "gc":
        holder.clear()
        import gc; gc.collect()
        torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
try:
    with torch.cuda.graph(graph):
        step()
        print("inside capture: status", torch.cuda.is_current_stream_capturing(), flush=True)
    graph.replay()
    torch.cuda.synchronize()
    print(variant, "ok", torch.equal(x, x_eager), holder["S"].stats()["iterations"])
except Exception as e:
    print(variant, "FAIL", str(e)[:200])
