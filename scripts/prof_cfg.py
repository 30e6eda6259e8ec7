"""Device time of one configs[i] grid build + solve vs the sum of its kernels' event times (is
the GPU busy or waiting on the host?): python scripts/prof_cfg.py c3"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1511_03296_b200 as fbs  # noqa: E402
from workloads import make  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
w = make(name)
dev = torch.device("cuda:0")
rgb, t, c = (torch.from_numpy(a).to(dev) for a in (w.rgb, w.t, w.c))
opts = dict(precond=w.precond, init=w.init, mode=w.mode, tol=w.tol, max_iters=w.max_iters, iters=w.iters)
pyr = w.precond == "hier" or w.init == "hier"


def run():
    g = fbs.grid_build(rgb, w.sigma_xy, w.sigma_l, w.sigma_uv, build_pyramid=pyr)
    fbs.solve(g, t, c, w.lam, **opts)
    g.close()


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    run()
e1.record()
torch.cuda.synchronize()
wall = e0.elapsed_time(e1) / 10
import time
torch.cuda.synchronize()
h0 = time.perf_counter()
for _ in range(10):
    run()
h1 = time.perf_counter()
torch.cuda.synchronize()
h2 = time.perf_counter()
print(f"host: {1e3 * (h1 - h0) / 10:.3f} ms per build+solve enqueued (incl. the build's syncs), "
      f"{1e3 * (h2 - h0) / 10:.3f} ms per build+solve to completion")
fbs.profile_reset()
fbs.profile_enable(True)
run()
torch.cuda.synchronize()
fbs.profile_enable(False)
rep = fbs.profile_report()
tot = sum(v[1] for v in rep.values())
n = sum(v[0] for v in rep.values())
print(f"{name}: wall {wall:.3f} ms per build+solve, {n} launches, summed kernel time {tot:.3f} ms")
for k, v in sorted(rep.items(), key=lambda kv: -kv[1][1])[:12]:
    print(f"  {k:36s} {v[0]:5d} {v[1]:.3f} ms  avg {1e3 * v[1] / v[0]:.1f} us")
