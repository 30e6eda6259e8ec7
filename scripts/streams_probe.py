"""Bench-step throughput with one compute stream vs steps alternating over S streams (a serving
pipeline with S steps in flight): python scripts/streams_probe.py [S ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1511_03296_b200 as fbs  # noqa: E402
from workloads import make  # noqa: E402

w = make("c5", frames=8)
dev = torch.device("cuda", 0)
main = torch.cuda.current_stream()


def run(nstreams, steps=40):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    bufs = [tuple(torch.from_numpy(a).to(dev) for a in (w.rgb, w.t, w.c)) + (torch.empty(w.t.shape, device=dev),)
            for _ in range(nstreams)]

    def go(n):
        ev = torch.cuda.Event()
        ev.record(main)
        for st in streams:
            st.wait_event(ev)
        for i in range(n):
            k = i % nstreams
            rgb, t, c, x = bufs[k]
            with torch.cuda.stream(streams[k]):
                g = fbs.grid_build(rgb, 8.0, 4.0, 3.0, n_bistoch=20)
                fbs.solve(g, t, c, 128.0, precond="hier", init="hier", mode="fixed", iters=25, out=x)
                g.close()
        for st in streams:
            main.wait_stream(st)

    go(2 * nstreams)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    go(steps)
    e1.record(main)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return ms, w.pixels / 1e6 / (ms / 1e3)


for rep in range(2):
    for s in [int(a) for a in sys.argv[1:]] or [1, 2, 3]:
        ms, mps = run(s)
        print(f"streams {s}: {ms:.3f} ms/step  {mps:.0f} MP/s", flush=True)
