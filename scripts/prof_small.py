"""One Jacobi TOL solve each of configs[0] (one-CTA path, k_pcg_small) and configs[3] (cluster
path, k_pcg_cluster) for ncu:  ncu --set full -k regex:k_pcg_ python scripts/prof_small.py"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1511_03296_b200 as fbs  # noqa: E402
from workloads import make  # noqa: E402

for name in ("c1", "c4"):
    w = make(name)
    rgb, t, c = (torch.from_numpy(a).cuda() for a in (w.rgb, w.t, w.c))
    g = fbs.grid_build(rgb, w.sigma_xy, w.sigma_l, w.sigma_uv, n_bistoch=w.n_bistoch)
    fbs.solve(g, t, c, w.lam, precond="jacobi", init="flat", mode="tol", tol=w.tol, max_iters=w.max_iters)
    torch.cuda.synchronize()
print("ok")
