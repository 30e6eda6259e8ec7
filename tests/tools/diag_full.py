"""Where does the full-size configs[4] frame-0 solution differ from the oracle? (diagnostic)"""
import os
import sys

import numpy as np
import torch

_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(_ROOT, "tests"))
sys.path.insert(0, _ROOT)
import oracle as O  # noqa: E402
import paper_1511_03296_b200 as fbs  # noqa: E402
from parity_util import oracle_opts, target_range, zero_conf_pixels  # noqa: E402
from workloads import make  # noqa: E402

w = make("c5", frames=1)
HW = w.H * w.W
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
og, sols = O.solve(w.rgb, w.t, w.c, w.sigma_xy, w.sigma_l, w.sigma_uv, w.lam, oracle_opts(w))
sol = sols[0]
rng = target_range(w.t[0].reshape(1, HW), w.c[0].ravel())[0]
zc = zero_conf_pixels(sol)
for mode, iters in (("fixed", 25), ("fixed", 60), ("tol", 0)):
    g = fbs.grid_build(dev(w.rgb), w.sigma_xy, w.sigma_l, w.sigma_uv)
    kw = dict(precond="hier", init="hier", mode=mode, iters=iters, tol=1e-6, max_iters=2000)
    x = fbs.solve(g, dev(w.t), dev(w.c), w.lam, **kw).cpu().numpy()[0].reshape(HW)
    o = O.solve(w.rgb, w.t, w.c, w.sigma_xy, w.sigma_l, w.sigma_uv, w.lam,
                oracle_opts(w, mode=mode, iters=iters, tol=1e-6))[1][0]
    d = np.abs(x - o.x[0]) / rng
    d[zc] = 0
    bad = np.nonzero(d > 1e-3)[0]
    print(mode, iters, "max", d.max(), "rms", np.sqrt(np.mean(d ** 2)), "n>1e-3", bad.size, "oracle iters",
          o.iterations)
    if bad.size:
        v = o.vid[bad]
        print("  bad vertices", np.unique(v).size, "Sc", o.sys.Sc[np.unique(v)][:8], "c", w.c[0].ravel()[bad][:8])
        print("  x gpu", x[bad][:5], "oracle", o.x[0][bad][:5], "t", w.t[0].ravel()[bad][:5])
    g.close()
