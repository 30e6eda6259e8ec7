"""Domain-transform post-filter on the bench workload's 8 × 1920×1080 frames (ncu target)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1511_03296_b200 as fbs  # noqa: E402
from workloads import make  # noqa: E402

w = make("c5", frames=8)
rgb, t = torch.from_numpy(w.rgb).cuda(), torch.from_numpy(w.t).cuda()
y = fbs.dt_filter(rgb, t, 16.0, 16.0)
torch.cuda.synchronize()
print("ok", float(y.mean()))
