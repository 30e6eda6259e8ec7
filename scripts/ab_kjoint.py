"""A/B of the K > 1 SpMV (FBS_SPMV_K=joint|split) on configs[3] (K = 21) and on 2 bench frames
with 21 channels: python scripts/ab_kjoint.py"""
import os
import subprocess
import sys

CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1511_03296_b200 as fbs
from workloads import make
dev = torch.device('cuda:0')
def ms(fn, n=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
w = make('c4')
rgb, t, c = (torch.from_numpy(a).to(dev) for a in (w.rgb, w.t, w.c))
g = fbs.grid_build(rgb, w.sigma_xy, w.sigma_l, w.sigma_uv)
a = ms(lambda: fbs.solve(g, t, c, w.lam, precond='jacobi', init='flat', mode='fixed', iters=25))
b = ms(lambda: fbs.solve(g, t, c, w.lam, precond='hier', init='hier', mode='fixed', iters=25))
w2 = make('c5', frames=2)
t21 = torch.from_numpy(np.repeat(w2.t, 21, axis=1)).to(dev)
g2 = fbs.grid_build(torch.from_numpy(w2.rgb).to(dev), 8.0, 4.0, 3.0)
c2 = torch.from_numpy(w2.c).to(dev)
d = ms(lambda: fbs.solve(g2, t21, c2, 128.0, precond='hier', init='hier', mode='fixed', iters=25), n=2)
prof = fbs.profile_enable(True); fbs.profile_reset()
fbs.solve(g, t, c, w.lam, precond='jacobi', init='flat', mode='fixed', iters=25); torch.cuda.synchronize()
r = fbs.profile_report(); fbs.profile_enable(False)
sp = {k: round(1e3 * v[1] / v[0], 1) for k, v in r.items() if 'spmv' in k}
print(f"c4 jacobi fixed25 {a:.3f} ms, c4 hier fixed25 {b:.3f} ms, 2x1080p K=21 hier fixed25 {d:.2f} ms, spmv avg us {sp}")
"""

for mode in ("joint", "split", "joint", "split"):
    env = dict(os.environ, FBS_SPMV_K=mode)
    out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print(mode, out.stdout.strip() or out.stderr[-800:])
