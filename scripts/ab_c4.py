"""A/B timing of configs[3] (K = 21) solves: python scripts/ab_c4.py [lib.so ...] (FBS_LIB per run)."""
import json
import os
import subprocess
import sys

CHILD = r"""
import json, sys, torch
sys.path.insert(0, '.')
import paper_1511_03296_b200 as fbs
from workloads import make
dev = torch.device('cuda:0')
w = make('c4')
rgb, t, c, gg = (torch.from_numpy(a).to(dev) for a in (w.rgb, w.t, w.c, w.g))
g = fbs.grid_build(rgb, w.sigma_xy, w.sigma_l, w.sigma_uv, n_bistoch=w.n_bistoch)
def ms(fn, n=7):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
def jac():
    x, S = fbs.solve(g, t, c, w.lam, precond='jacobi', init='flat', mode='tol', tol=1e-6, keep_system=True)
    S.backward(gg, t, c)
    return S
S = jac()
it = S.stats()['iterations']
out = {'jacobi_fwd_bwd_ms': ms(jac), 'jacobi_iters_max': int(it.max()),
       'hier_full_ms': ms(lambda: fbs.solve(g, t, c, w.lam, precond='hier', init='hier', mode='tol', tol=1e-6)),
       'hier_lowrank_ms': ms(lambda: fbs.solve(g, t, c, w.lam, precond='hier', init='hier', mode='tol', tol=1e-6, lowrank_eps=0.01))}
print(json.dumps(out))
"""

libs = sys.argv[1:] or [""]
for rep in range(3):
    for lib in libs:
        env = dict(os.environ)
        if lib:
            env["FBS_LIB"] = os.path.abspath(lib)
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-2000:]
        print(lib or "default", line, flush=True)
