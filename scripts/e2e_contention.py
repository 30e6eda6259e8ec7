"""Does host<->device DMA slow the bench step?  Device time of K bench steps alone, then with
independent H2D (and D2H) copies of the step's input (output) size running on side streams the
whole time: python scripts/e2e_contention.py [K]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1511_03296_b200 as fbs  # noqa: E402
from workloads import make  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
w = make("c5")
dev = torch.device("cuda", 0)
rgb, t, c = (torch.from_numpy(a).to(dev) for a in (w.rgb, w.t, w.c))
x = torch.empty_like(t)
h_in = torch.empty(182_476_800, dtype=torch.uint8).pin_memory()
d_in = torch.empty(182_476_800, dtype=torch.uint8, device=dev)
h_out = torch.empty(66_355_200, dtype=torch.uint8).pin_memory()
d_out = torch.empty(66_355_200, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def step():
    g = fbs.grid_build(rgb, 8.0, 4.0, 3.0, n_bistoch=20)
    fbs.solve(g, t, c, 128.0, precond="hier", init="hier", mode="fixed", iters=25, out=x)
    g.close()


def timed(copies):
    torch.cuda.synchronize()
    if copies:
        for _ in range(2 * K):  # more than enough copies to cover the K steps
            with torch.cuda.stream(s1):
                d_in.copy_(h_in, non_blocking=True)
            if copies > 1:
                with torch.cuda.stream(s2):
                    h_out.copy_(d_out, non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        step()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K


for _ in range(3):
    step()
for r in range(2):
    print("alone %.3f ms  with H2D %.3f ms  with H2D+D2H %.3f ms" % (timed(0), timed(1), timed(2)))
