"""Per-kernel launch times of the PCG with ONE frame group (FBS_PCG_GROUPS=1 set here), so each
launch has the GPU to itself: `python scripts/spmv_iso.py [frames] [kernel prefixes,...]`.
Same-box A/B: FBS_LIB=other.so python scripts/spmv_iso.py 4."""
import os
import sys

os.environ.setdefault("FBS_PCG_GROUPS", "1")
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1511_03296_b200 as fbs  # noqa: E402
from workloads import make  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 4
want = (sys.argv[2] if len(sys.argv) > 2 else "k_spmv2,k_hier_level0<UPDATE>,k_tree_lift<PCG>,k_tree_coarse<PCG>,k_tree_level0<PCG>").split(",")
dev = torch.device("cuda", 0)
w = make("c5", frames=frames, first_frame=0)
rgb, t, c = (torch.from_numpy(a).to(dev) for a in (w.rgb, w.t, w.c))
g = fbs.grid_build(rgb, 8.0, 4.0, 3.0, n_bistoch=20)
for _ in range(2):
    fbs.solve(g, t, c, 128.0, precond="hier", init="hier", mode="fixed", iters=25)
torch.cuda.synchronize()
fbs.profile_enable(True)
fbs.profile_reset()
for _ in range(5):
    fbs.solve(g, t, c, 128.0, precond="hier", init="hier", mode="fixed", iters=25)
torch.cuda.synchronize()
rep = fbs.profile_report()
fbs.profile_enable(False)
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    fbs.solve(g, t, c, 128.0, precond="hier", init="hier", mode="fixed", iters=25)
e1.record()
torch.cuda.synchronize()
out = " ".join("%s=%.2f" % (k, 1e3 * ms / n) for k, (n, ms) in rep.items() if any(k.startswith(p) for p in want))
print("M=%d solve_ms=%.3f %s" % (g.M, e0.elapsed_time(e1) / 10, out))
