# configs[4] to tol 1e-6 (8 frames) under environment settings: bash scripts/ab_c5tol.sh "VAR=a VAR=b"
for kv in $1; do
env $kv python -c "
import torch, sys
sys.path.insert(0,'.')
import paper_1511_03296_b200 as fbs
from workloads import make
w = make('c5')
rgb, t, c = (torch.from_numpy(a).cuda() for a in (w.rgb, w.t, w.c))
g = fbs.grid_build(rgb, 8.0, 4.0, 3.0)
run = lambda: fbs.solve(g, t, c, 128.0, precond='hier', init='hier', mode='tol', tol=1e-6)
for _ in range(2): run()
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run(); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
print('$kv', round(best, 3))
"
done
