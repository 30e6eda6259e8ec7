"""One profiled bench step with FBS_TIMELINE set: prints the PCG iteration's per-stream kernel
timeline (start, duration) for overlap analysis.  python scripts/timeline.py [csv path]"""
import csv
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/timeline.csv"
os.environ["FBS_TIMELINE"] = path
import paper_1511_03296_b200 as fbs  # noqa: E402
from workloads import make  # noqa: E402

w = make("c5")
rgb, t, c = (torch.from_numpy(a).cuda() for a in (w.rgb, w.t, w.c))
x = torch.empty_like(t)
for _ in range(3):
    g = fbs.grid_build(rgb, 8.0, 4.0, 3.0)
    fbs.solve(g, t, c, 128.0, precond="hier", init="hier", mode="fixed", iters=25, out=x)
    g.close()
torch.cuda.synchronize()
fbs.profile_reset()
fbs.profile_enable(True)
g = fbs.grid_build(rgb, 8.0, 4.0, 3.0)
fbs.solve(g, t, c, 128.0, precond="hier", init="hier", mode="fixed", iters=25, out=x)
g.close()
torch.cuda.synchronize()
fbs.profile_enable(False)
fbs.profile_report()
rows = list(csv.DictReader(open(path)))
streams = {}
for r in rows:
    streams.setdefault(r["stream"], len(streams))
pcg = [r for r in rows if r["name"] in ("k_spmv2", "k_hier_level0<UPDATE>", "k_tree_lift<PCG>", "k_tree_coarse<PCG>",
                                         "k_tree_level0<PCG>")]
t0 = float(pcg[20]["start_us"]) if len(pcg) > 40 else 0.0
for r in sorted(pcg, key=lambda r: float(r["start_us"]))[20:40]:
    print(f"s{streams[r['stream']]} {float(r['start_us']) - t0:9.1f} +{float(r['dur_us']):6.1f}  {r['name']}")
