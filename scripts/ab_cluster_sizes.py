"""Device ms per Jacobi TOL solve (build excluded) over frame sizes and channel counts, with the
one-launch paths on and off (FBS_SMALL_PX / FBS_CLUSTER_PX read once per process, so one child per
setting, interleaved):  python scripts/ab_cluster_sizes.py"""
import json
import os
import subprocess
import sys

CHILD = r"""
import json, sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_1511_03296_b200 as fbs
from workloads.synth import voronoi_reference
out = {}
for (H, W) in ((96, 128), (150, 200), (240, 320), (375, 500), (480, 640)):
    for K in (1, 3, 21):
        rng = np.random.default_rng(H + K)
        rgb = torch.from_numpy(voronoi_reference(rng, W, H, 30, "gradient", 3.0)[0][None].copy()).cuda()
        t = torch.from_numpy(rng.uniform(0, 10, (1, K, H, W)).astype(np.float32)).cuda()
        c = torch.from_numpy(rng.uniform(0.1, 1, (1, H, W)).astype(np.float32)).cuda()
        g = fbs.grid_build(rgb, 8.0, 4.0, 3.0)
        run = lambda: fbs.solve(g, t, c, 128.0, precond="jacobi", init="flat", mode="tol", tol=1e-6, max_iters=5000)
        for _ in range(3): run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(5):
            e0.record(); run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        out[f"{H}x{W}xK{K}"] = round(sorted(ts)[2], 3)
print(json.dumps(out))
"""
res = {}
for rnd in range(2):
    for name, env in (("multi", {"FBS_SMALL_PX": "0", "FBS_CLUSTER_PX": "0"}), ("cluster", {"FBS_SMALL_PX": "0", "FBS_CLUSTER_PX": "1000000"}),
                      ("small", {"FBS_SMALL_PX": "1000000", "FBS_CLUSTER_PX": "0"})):
        p = subprocess.run([sys.executable, "-c", CHILD], env=dict(os.environ, **env), capture_output=True, text=True)
        d = json.loads(p.stdout.strip().splitlines()[-1]) if p.returncode == 0 else {"err": p.stderr[-400:]}
        print(rnd, name, json.dumps(d), flush=True)
