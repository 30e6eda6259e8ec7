"""Per-kernel event times of the domain-transform post-filter on the bench frames (8 × 1920×1080):
python scripts/prof_dt_events.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1511_03296_b200 as fbs  # noqa: E402
from workloads import make  # noqa: E402

w = make("c5", frames=8)
rgb, t = torch.from_numpy(w.rgb).cuda(), torch.from_numpy(w.t).cuda()
out = torch.empty_like(t)
for _ in range(3):
    fbs.dt_filter(rgb, t, 16.0, 16.0, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    fbs.dt_filter(rgb, t, 16.0, 16.0, out=out)
e1.record()
torch.cuda.synchronize()
print(f"dt_filter: {e0.elapsed_time(e1) / 10:.3f} ms per call")
fbs.profile_reset()
fbs.profile_enable(True)
fbs.dt_filter(rgb, t, 16.0, 16.0, out=out)
torch.cuda.synchronize()
fbs.profile_enable(False)
for k, v in sorted(fbs.profile_report().items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:24s} {v[0]:3d} {v[1]:.3f} ms  avg {1e3 * v[1] / v[0]:.1f} us")
