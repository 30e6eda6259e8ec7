import torch, sys
sys.path.insert(0, '.')
import paper_1511_03296_b200 as fbs
from workloads import make
w = make('c5')
rgb, t, c = (torch.from_numpy(a).cuda() for a in (w.rgb, w.t, w.c))
x = torch.empty_like(t)
for i in range(6):
    g = fbs.grid_build(rgb, 8.0, 4.0, 3.0)
    fbs.solve(g, t, c, 128.0, precond='hier', init='hier', mode='fixed', iters=25, out=x)
    g.close()
    print('--- step', i, file=sys.stderr)
torch.cuda.synchronize()
