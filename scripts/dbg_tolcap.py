"""DEBUG: capture a TOL solve into a CUDA graph: grid built inside/outside, system kept or not."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1511_03296_b200 as fbs
from workloads import make

w = make("c5", frames=1, W=200, H=120, n_cells=16)
dev = torch.device("cuda")
rgb, t, c = (torch.from_numpy(a).to(dev) for a in (w.rgb, w.t, w.c))
x = torch.empty_like(t)
kw = dict(precond="hier", init="hier", mode="tol", tol=1e-6, max_iters=500)
g0 = fbs.grid_build(rgb, w.sigma_xy, w.sigma_l, w.sigma_uv)
torch.cuda.synchronize()
for inside in (False, True):
    for keep in (False, True):
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                g = fbs.grid_build(rgb, w.sigma_xy, w.sigma_l, w.sigma_uv) if inside else g0
                r = fbs.solve(g, t, c, w.lam, out=x, keep_system=keep, **kw)
            graph.replay()
            torch.cuda.synchronize()
            print(inside, keep, "ok", float(x.mean()), flush=True)
        except Exception as e:
            print(inside, keep, "FAIL", str(e)[:200], flush=True)
            try:
                torch.cuda.synchronize()
            except Exception as e2:
                print("  sync:", str(e2)[:100])
