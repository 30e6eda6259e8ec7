"""TOL-mode single-frame solves (configs[0], [1], [3]) under environment variants:
python scripts/ab_tol.py  (FBS_TOL_CHUNK, FBS_TOL_GRAPH)"""
import os
import subprocess
import sys

CHILD = r"""
import sys, torch
sys.path.insert(0, '.')
import paper_1511_03296_b200 as fbs
from workloads import make
dev = torch.device('cuda:0')
out = []
for name in ('c1', 'c2', 'c4'):
    w = make(name)
    rgb, t, c = (torch.from_numpy(a).to(dev) for a in (w.rgb, w.t, w.c))
    pyr = w.precond == 'hier' or w.init == 'hier'
    g = fbs.grid_build(rgb, w.sigma_xy, w.sigma_l, w.sigma_uv, build_pyramid=pyr)
    run = lambda: fbs.solve(g, t, c, w.lam, precond=w.precond, init=w.init, mode='tol', tol=1e-6)
    for _ in range(3): run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): run()
    e1.record(); torch.cuda.synchronize()
    out.append(f"{name} {e0.elapsed_time(e1) / 10:.3f}")
print(' '.join(out))
"""
for env in ("", "FBS_TOL_CHUNK=4", "FBS_TOL_CHUNK=2", "FBS_TOL_CHUNK=16", "FBS_TOL_GRAPH=1"):
    e = dict(os.environ)
    if env:
        k, v = env.split("=")
        e[k] = v
    r = subprocess.run([sys.executable, "-c", CHILD], env=e, capture_output=True, text=True)
    print(env or "default", r.stdout.strip() or r.stderr[-500:])
