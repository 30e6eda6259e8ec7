"""Bug hunt (test infrastructure: runs the oracle): the seeded random cases of
tests/test_gpu_random.py over many more seeds — grid bit-exactness and TOL solve parity (hier and
Jacobi).  python tests/tools/fuzz_random.py FIRST COUNT"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_1511_03296_b200 as fbs  # noqa: E402
from parity_util import MAX_TOL, RMS_TOL, compare_x, zero_conf_pixels  # noqa: E402
from test_gpu_random import case  # noqa: E402

first, count = int(sys.argv[1]), int(sys.argv[2])
bad = 0
for seed in range(first, first + count):
    rgb, t, c, sig, lam = case(seed)
    F, H, W = rgb.shape[:3]
    K, HW = t.shape[1], H * W
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    g = fbs.grid_build(d(rgb), *sig)
    og = O.build_grid(rgb, *sig)
    e = g.export()
    msg = []
    if g.M != og.M or any(not np.array_equal(e[k], getattr(og, k)) for k in ("keys", "vid", "m", "nbr")):
        msg.append("grid")
    for pc in ("hier+hier", "jacobi+flat"):
        p, i = pc.split("+")
        x = fbs.solve(g, d(t), d(c), lam, precond=p, init=i, mode="tol", tol=1e-6, max_iters=5000).cpu().numpy()
        _, sols = O.solve(rgb, t, c, *sig, lam, O.SolveOptions(precond=p, init=i, mode="tol", tol=1e-6, max_iters=5000))
        for f, sol in enumerate(sols):
            mx, rms = compare_x(x[f].reshape(K, HW), sol.x, t[f].reshape(K, HW).astype(np.float64),
                                c[f].reshape(HW).astype(np.float64), exclude=zero_conf_pixels(sol))
            if not (mx <= MAX_TOL and rms <= RMS_TOL):
                msg.append(f"{pc} f{f} max {mx:.2e} rms {rms:.2e}")
    g.close()
    if msg:
        bad += 1
        print(seed, (F, K, H, W), sig, lam, "; ".join(msg), flush=True)
print(f"{count - bad}/{count} seeds clean")
