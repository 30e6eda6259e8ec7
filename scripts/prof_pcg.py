"""One hierarchical solve of the bench workload (configs[4], 8 × 1920×1080 frames) with a few PCG
iterations: the target of `ncu -k regex:k_tile ...` captures."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1511_03296_b200 as fbs  # noqa: E402
from workloads import make  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 4
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dev = torch.device("cuda", 0)
w = make("c5", frames=frames, first_frame=0)
rgb, t, c = (torch.from_numpy(a).to(dev) for a in (w.rgb, w.t, w.c))
g = fbs.grid_build(rgb, 8.0, 4.0, 3.0, n_bistoch=20)
x = fbs.solve(g, t, c, 128.0, precond="hier", init="hier", mode="fixed", iters=iters)
torch.cuda.synchronize()
print("ok", g.M, g.info())
