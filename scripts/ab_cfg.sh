# configs[0..3] device times under environment settings: bash scripts/ab_cfg.sh "VAR=a VAR=b ..."
for r in 1 2; do for kv in $1; do
env $kv python -c "
import torch, sys, json
sys.path.insert(0, '.')
import paper_1511_03296_b200 as fbs
from workloads import make
out = {}
for name in ('c1', 'c2', 'c3', 'c4'):
    w = make(name)
    rgb, t, c = (torch.from_numpy(a).cuda() for a in (w.rgb, w.t, w.c))
    gg = torch.from_numpy(w.g).cuda() if w.g is not None else None
    opts = dict(precond=w.precond, init=w.init, mode=w.mode, tol=w.tol, max_iters=w.max_iters, iters=w.iters)
    def run():
        g = fbs.grid_build(rgb, w.sigma_xy, w.sigma_l, w.sigma_uv)
        if gg is not None:
            _, S = fbs.solve(g, t, c, w.lam, keep_system=True, **opts); S.backward(gg, t, c); S.close()
        else:
            fbs.solve(g, t, c, w.lam, **opts)
        g.close()
    for _ in range(2): run()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); run(); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    out[name] = round(best, 3)
print('$kv', out)
"
done; done
