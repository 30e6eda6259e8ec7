"""The one-launch Jacobi PCG for small frames (k_pcg_small: one CTA; k_pcg_cluster: a cluster of 8
CTAs per (frame, channel); api.cu run_pcg) against the oracle and against the multi-kernel path of
the same library (FBS_SMALL_PX=0 FBS_CLUSTER_PX=0, in a subprocess: the bounds are read once per
process).  Same per-vertex arithmetic and stopping rule (Alg. 2;
reading #11); only the fp64 dot products' summation order differs, so the two paths agree to
fp32 rounding and stop within one iteration of each other.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
from parity_util import MAX_TOL, RMS_TOL, compare_x, oracle_opts, zero_conf_pixels
from workloads import make

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1511_03296_b200 as fbs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = {
    "c1": dict(name="c1", kw={}),                                              # configs[0]: 48x64
    "c5_3f": dict(name="c5", kw=dict(frames=3, W=120, H=96, n_cells=12)),      # 3 small frames
    "c4_k": dict(name="c4", kw=dict(W=100, H=75, n_cells=8)),                  # K > 1 channels
    # > 8192 px: the cluster path (k_pcg_cluster, 8 CTAs per (frame, channel))
    "c5_mid": dict(name="c5", kw=dict(frames=2, W=320, H=240, n_cells=30)),
    "c4_mid": dict(name="c4", kw=dict(W=300, H=225, n_cells=16)),
}
MODES = {
    "tol": dict(precond="jacobi", init="flat", mode="tol", tol=1e-6, max_iters=5000),
    "fixed": dict(precond="jacobi", init="flat", mode="fixed", iters=25),
    "zero_tol": dict(precond="jacobi", init="zero", mode="tol", tol=1e-6, max_iters=5000),
}


def _solve(case, mode, backward=False):
    c = CASES[case]
    w = make(c["name"], **c["kw"])
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    g = fbs.grid_build(dev(w.rgb), w.sigma_xy, w.sigma_l, w.sigma_uv, n_bistoch=w.n_bistoch)
    t, cc = dev(w.t), dev(w.c)
    n0 = fbs.launch_count()
    x, S = fbs.solve(g, t, cc, w.lam, keep_system=True, **MODES[mode])
    torch.cuda.synchronize()
    n1 = fbs.launch_count()
    out = {"x": x.cpu().numpy(), "iters": np.asarray(S.stats()["iterations"]).tolist(), "launches": n1 - n0}
    if backward:
        dt, dc = S.backward(torch.ones_like(x), t, cc)
        out["dt"], out["dc"] = dt.cpu().numpy(), dc.cpu().numpy()
    return w, out


def _multi_kernel(case, mode, backward, out_path):
    code = (
        "import sys, numpy as np; sys.path.insert(0, 'tests'); "
        "import test_gpu_small as T; "
        f"w, o = T._solve({case!r}, {mode!r}, {backward!r}); "
        f"np.savez({str(out_path)!r}, **{{k: np.asarray(v) for k, v in o.items()}})"
    )
    env = dict(os.environ, FBS_SMALL_PX="0", FBS_CLUSTER_PX="0")
    subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, check=True, timeout=600)
    z = np.load(out_path)
    return {k: z[k] for k in z.files}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("mode", list(MODES))
def test_small_path_vs_oracle_and_multi_kernel(case, mode, tmp_path):
    w, one = _solve(case, mode, backward=(mode == "tol"))
    ref = _multi_kernel(case, mode, (mode == "tol"), tmp_path / "multi_kernel.npz")
    # the one-CTA path ran: 2 launches per solve (scalars + k_pcg_small) plus set-up, against
    # several per PCG iteration on the multi-kernel path
    assert one["launches"] < ref["launches"]
    it1, it0 = np.asarray(one["iters"]), np.asarray(ref["iters"])
    if mode == "fixed":
        assert np.array_equal(it1, it0)
    else:
        assert np.all(np.abs(it1 - it0) <= 1), (it1, it0)
    rng = float(w.t.max() - w.t.min()) or 1.0
    # fixed count: the iterate itself, not a converged solution, is compared (reading #29)
    assert np.max(np.abs(one["x"] - ref["x"])) <= (1e-3 if mode == "fixed" else 1e-4) * rng
    if "dt" in one:
        s = float(np.max(np.abs(ref["dt"]))) or 1.0
        assert np.max(np.abs(one["dt"] - ref["dt"])) <= 1e-4 * s
        # dL/dc is dL/dt-sized times (x − t)-sized; at a converged solve it is
        # near zero, so its scale is max|dL/dt| · range, not its own maximum
        s = float(np.max(np.abs(ref["dt"]))) * rng or 1.0
        assert np.max(np.abs(one["dc"] - ref["dc"])) <= 1e-4 * s
    # and the oracle (north_star's tolerances), frame by frame
    og, sols = O.solve(w.rgb, w.t, w.c, w.sigma_xy, w.sigma_l, w.sigma_uv, w.lam, oracle_opts(w, **MODES[mode]))
    HW = w.H * w.W
    for f, sol in enumerate(sols):
        t = w.t[f].reshape(w.K, HW).astype(np.float64)
        c = w.c[f].reshape(HW).astype(np.float64)
        mx, rms = compare_x(one["x"][f].reshape(w.K, HW), sol.x, t, c, exclude=zero_conf_pixels(sol))
        assert mx <= MAX_TOL and rms <= RMS_TOL, (f, mx, rms)
        if mode == "fixed":
            assert np.all(it1[f] == np.minimum(25, sol.iterations))
