"""Bench-workload step issued as S concurrent half-batches on S streams (frames are independent):
python scripts/ab_split.py — device ms per 8-frame step for S = 1, 2, 4."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1511_03296_b200 as fbs  # noqa: E402
from workloads import make  # noqa: E402

dev = torch.device("cuda:0")
w = make("c5")
rgb, t, c = (torch.from_numpy(a).to(dev) for a in (w.rgb, w.t, w.c))
x = torch.empty_like(t)


def step(S, streams):
    F = w.frames
    main = torch.cuda.current_stream()
    for i in range(S):
        f0, f1 = F * i // S, F * (i + 1) // S
        st = streams[i]
        st.wait_stream(main)
        with torch.cuda.stream(st):
            g = fbs.grid_build(rgb[f0:f1], 8.0, 4.0, 3.0)
            fbs.solve(g, t[f0:f1], c[f0:f1], 128.0, precond="hier", init="hier", mode="fixed", iters=25,
                      out=x[f0:f1])
            g.close()
    for st in streams[:S]:
        main.wait_stream(st)


streams = [torch.cuda.Stream() for _ in range(4)]
for S in (1, 2, 4, 1, 2, 4):
    for _ in range(3):
        step(S, streams)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        step(S, streams)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"S={S}: {ms:.3f} ms per step, {w.pixels / 1e3 / ms:.0f} MP/s")
