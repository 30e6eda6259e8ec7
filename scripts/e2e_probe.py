"""Which part of the end-to-end pipeline costs time: the bench step with/without its copies."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1511_03296_b200 as fbs  # noqa: E402
from workloads import make  # noqa: E402

w = make("c5", frames=8)
dev = torch.device("cuda", 0)
rgb_h, t_h, c_h = (torch.from_numpy(a).pin_memory() for a in (w.rgb, w.t, w.c))
x_h = torch.empty(t_h.shape, dtype=torch.float32).pin_memory()
stream = torch.cuda.current_stream()
s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
bufs = [tuple(a.to(dev) for a in (rgb_h, t_h, c_h)) + (torch.empty(t_h.shape, device=dev),) for _ in range(2)]
x_hs = [x_h, torch.empty_like(x_h).pin_memory()]


def step_on(rgb_b, t_b, c_b, x_b):
    g = fbs.grid_build(rgb_b, 8.0, 4.0, 3.0, n_bistoch=20)
    fbs.solve(g, t_b, c_b, 128.0, precond="hier", init="hier", mode="fixed", iters=25, out=x_b)
    g.close()


def run(n, do_h2d, do_d2h, ahead):
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_comp = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]

    def h2d(i):
        slot = i % 2
        with torch.cuda.stream(s_h2d):
            if i >= 2:
                s_h2d.wait_event(ev_comp[slot])
            if do_h2d:
                for d, h in zip(bufs[slot][:3], (rgb_h, t_h, c_h)):
                    d.copy_(h, non_blocking=True)
            ev_in[slot].record(s_h2d)

    if ahead:
        h2d(0)
    for i in range(n):
        slot = i % 2
        if ahead and i + 1 < n:
            h2d(i + 1)
        if not ahead:
            h2d(i)
        stream.wait_event(ev_in[slot])
        if i >= 2:
            stream.wait_event(ev_out[slot])
        step_on(*bufs[slot])
        ev_comp[slot].record(stream)
        with torch.cuda.stream(s_d2h):
            s_d2h.wait_event(ev_comp[slot])
            if do_d2h:
                x_hs[slot].copy_(bufs[slot][3], non_blocking=True)
            ev_out[slot].record(s_d2h)
    stream.wait_event(ev_out[(n - 1) % 2])
    stream.wait_event(ev_out[(n - 2) % 2])


def timed(**kw):
    run(3, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s_h2d.wait_event(e0)
    run(20, **kw)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 20


for rep in range(2):
    for name, kw in (("none", dict(do_h2d=False, do_d2h=False, ahead=False)),
                     ("h2d", dict(do_h2d=True, do_d2h=False, ahead=False)),
                     ("d2h", dict(do_h2d=False, do_d2h=True, ahead=False)),
                     ("both", dict(do_h2d=True, do_d2h=True, ahead=False)),
                     ("both_ahead", dict(do_h2d=True, do_d2h=True, ahead=True)),
                     ("h2d_ahead", dict(do_h2d=True, do_d2h=False, ahead=True))):
        print(name, round(timed(**kw), 3), flush=True)

# compute alone while a side stream streams copies continuously (no dependencies between them)
big_h = torch.empty(182_476_800, dtype=torch.uint8).pin_memory()
big_d = torch.empty(182_476_800, dtype=torch.uint8, device=dev)
out_h = torch.empty(66_355_200, dtype=torch.uint8).pin_memory()
out_d = torch.empty(66_355_200, dtype=torch.uint8, device=dev)
for mode in ("h2d", "d2h"):
    torch.cuda.synchronize()
    with torch.cuda.stream(s_h2d):
        for _ in range(40 if mode == "h2d" else 120):
            if mode == "h2d":
                big_d.copy_(big_h, non_blocking=True)
            else:
                out_h.copy_(out_d, non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        step_on(*bufs[0])
    e1.record()
    torch.cuda.synchronize()
    print("compute with background", mode, round(e0.elapsed_time(e1) / 10, 3), flush=True)

# per-kernel event times with and without a background D2H stream
for mode in ("none", "d2h"):
    torch.cuda.synchronize()
    if mode == "d2h":
        with torch.cuda.stream(s_h2d):
            for _ in range(120):
                out_h.copy_(out_d, non_blocking=True)
    fbs.profile_reset()
    fbs.profile_enable(True)
    for _ in range(10):
        step_on(*bufs[0])
    torch.cuda.synchronize()
    fbs.profile_enable(False)
    prof = fbs.profile_report()
    tot = sum(v[1] for v in prof.values()) / 10
    top = sorted(prof.items(), key=lambda kv: -kv[1][1])[:8]
    print("profile", mode, round(tot, 3), " ".join(f"{k}={v[1] / 10:.3f}" for k, v in top), flush=True)
