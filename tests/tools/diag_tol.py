"""Diagnostic: GPU vs oracle solutions at several stopping tolerances (ill-conditioned c3s)."""
import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle as O
import paper_1511_03296_b200 as fbs
from workloads import make
from parity_util import compare_x, zero_conf_pixels
name = sys.argv[1] if len(sys.argv) > 1 else 'c3s'
W = {'c3s': lambda: make('c3', H=272, W=344, n_cells=40), 'c2s': lambda: make('c2', W=347, H=277, n_cells=40),
     'c4s': lambda: make('c4', W=250, H=187, n_cells=20)}[name]()
HW = W.H*W.W
t = W.t[0].reshape(W.K, HW).astype(float); c = W.c[0].reshape(HW).astype(float)
for pc in ['jacobi+flat', 'hier+hier']:
    p, i = pc.split('+')
    ors = {}
    for tol in [1e-6, 1e-8, 1e-11]:
        og, sols = O.solve(W.rgb, W.t, W.c, W.sigma_xy, W.sigma_l, W.sigma_uv, W.lam, O.SolveOptions(precond=p, init=i, mode='tol', tol=tol, max_iters=20000))
        ors[tol] = sols[0]
    zc = zero_conf_pixels(ors[1e-6])
    g = fbs.grid_build(torch.from_numpy(W.rgb).cuda(), W.sigma_xy, W.sigma_l, W.sigma_uv)
    for tol in [1e-6, 1e-7, 1e-8]:
        x, s = fbs.solve(g, torch.from_numpy(W.t).cuda(), torch.from_numpy(W.c).cuda(), W.lam, keep_system=True, precond=p, init=i, mode='tol', tol=tol, max_iters=20000)
        xg = x.cpu().numpy()[0].reshape(W.K, HW)
        st = s.stats()
        # true residual of GPU y in fp64 with the oracle's A
        y = s.export()['y'].astype(float)
        A = ors[1e-11].sys.A; b = ors[1e-11].sys.b
        tr = np.linalg.norm(b - A @ y, axis=0) / np.linalg.norm(b, axis=0)
        for otol, so in ors.items():
            mx, rms = compare_x(xg, so.x, t, c, exclude=zc)
            print(f'{pc} gpu_tol={tol:g} it={st["iterations"].ravel()[:3]} rec={st["relres"].ravel()[:1]} true={tr[:1]} | oracle_tol={otol:g} it={so.iterations[:3]} max={mx:.3e} rms={rms:.3e}')
    for otol, so in ors.items():
        mx, rms = compare_x(so.x, ors[1e-11].x, t, c, exclude=zc)
        print(f'  oracle tol {otol:g} vs oracle 1e-11: max={mx:.3e} rms={rms:.3e}')
