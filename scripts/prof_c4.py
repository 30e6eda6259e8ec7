"""One configs[3] solve (K = 21) + backward: target of ncu launch lists.
python scripts/prof_c4.py [jacobi|hier]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1511_03296_b200 as fbs  # noqa: E402
from workloads import make  # noqa: E402

pc = sys.argv[1] if len(sys.argv) > 1 else "jacobi"
dev = torch.device("cuda", 0)
w = make("c4")
rgb, t, c, gg = (torch.from_numpy(a).to(dev) for a in (w.rgb, w.t, w.c, w.g))
g = fbs.grid_build(rgb, w.sigma_xy, w.sigma_l, w.sigma_uv, n_bistoch=w.n_bistoch)
init = "flat" if pc == "jacobi" else "hier"
x, S = fbs.solve(g, t, c, w.lam, precond=pc, init=init, mode="tol", tol=1e-6, keep_system=True)
S.backward(gg, t, c)
torch.cuda.synchronize()
print("ok", g.M, S.stats()["iterations"].max())
