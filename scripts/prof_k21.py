"""configs[3] (K = 21) hierarchical solve to tol 1e-6: wall time and per-kernel event times
(python scripts/prof_k21.py; FBS_LIB selects the library)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1511_03296_b200 as fbs  # noqa: E402
from workloads import make  # noqa: E402

w = make("c4")
dev = torch.device("cuda:0")
rgb, t, c = (torch.from_numpy(a).to(dev) for a in (w.rgb, w.t, w.c))
g = fbs.grid_build(rgb, w.sigma_xy, w.sigma_l, w.sigma_uv)


def run():
    fbs.solve(g, t, c, w.lam, precond="hier", init="hier", mode="tol", tol=1e-6)


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    run()
e1.record()
torch.cuda.synchronize()
print(f"wall {e0.elapsed_time(e1) / 5:.3f} ms")
fbs.profile_reset()
fbs.profile_enable(True)
run()
torch.cuda.synchronize()
fbs.profile_enable(False)
for k, v in sorted(fbs.profile_report().items(), key=lambda kv: -kv[1][1])[:10]:
    print(f"  {k:36s} {v[0]:5d} {v[1]:.3f} ms  avg {1e3 * v[1] / v[0]:.1f} us")
