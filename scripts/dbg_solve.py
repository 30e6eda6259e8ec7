import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1511_03296_b200 as fbs
from workloads import make
w = make(sys.argv[1] if len(sys.argv) > 1 else 'c2')
dev = torch.device('cuda:0')
rgb, t, c = (torch.from_numpy(a).to(dev) for a in (w.rgb, w.t, w.c))
g = fbs.grid_build(rgb, w.sigma_xy, w.sigma_l, w.sigma_uv)
torch.cuda.synchronize(); print('built', g.M, g.levels, flush=True)
for mode in ('fixed', 'tol'):
    x = fbs.solve(g, t, c, w.lam, precond=w.precond, init=w.init, mode=mode, tol=1e-6, iters=25)
    torch.cuda.synchronize(); print(mode, 'ok', float(x.mean()), flush=True)
