"""Device ms per grid build + solve of configs[0..3] (as bench.py's extras run them, plus configs[2]
to tol 1e-6) under (library, environment) variants, interleaved on one box:
  python scripts/ab_cfgs.py "lib.so:VAR=a,VAR2=b" "lib2.so:" ...
"""
import os
import subprocess
import sys

CHILD = r"""
import dataclasses, sys, torch
sys.path.insert(0, '.')
import paper_1511_03296_b200 as fbs
from workloads import make
dev = torch.device('cuda:0')
out = []
for name, over in (('c1', {}), ('c2', {}), ('c3', {}), ('c3_tol', {'mode': 'tol', 'max_iters': 5000}), ('c4', {})):
    w = make(name.split('_')[0])
    if over:
        w = dataclasses.replace(w, **over)
    rgb, t, c = (torch.from_numpy(a).to(dev) for a in (w.rgb, w.t, w.c))
    gq = torch.from_numpy(w.g).to(dev) if w.g is not None else None
    opts = dict(precond=w.precond, init=w.init, mode=w.mode, tol=w.tol, max_iters=w.max_iters)
    if w.mode == 'fixed':
        opts['iters'] = w.iters
    pyr = w.precond == 'hier' or w.init == 'hier'
    def run():
        g = fbs.grid_build(rgb, w.sigma_xy, w.sigma_l, w.sigma_uv, n_bistoch=w.n_bistoch, build_pyramid=pyr)
        if gq is not None:
            _, S = fbs.solve(g, t, c, w.lam, keep_system=True, **opts)
            S.backward(gq, t, c)
            S.close()
        else:
            fbs.solve(g, t, c, w.lam, **opts)
        g.close()
    reps = 3 if name == 'c3_tol' else 10
    for _ in range(3): run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): run()
    e1.record(); torch.cuda.synchronize()
    out.append(f"{name}={e0.elapsed_time(e1) / reps:.3f}")
print(' '.join(out))
"""

for r in range(2):
    for spec in sys.argv[1:]:
        lib, _, envs = spec.partition(":")
        e = dict(os.environ)
        if lib:
            e["FBS_LIB"] = os.path.abspath(lib)
        for kv in filter(None, envs.split(",")):
            k, _, v = kv.partition("=")
            e[k] = v
        res = subprocess.run([sys.executable, "-c", CHILD], env=e, capture_output=True, text=True)
        print(spec, res.stdout.strip() or res.stderr.strip()[-400:], flush=True)
