"""GPU parity of the robust bilateral solver (Supp. Alg. 3, fbs_solve_robust) against the oracle,
plus its edge cases and the robustness property at a larger size."""
import numpy as np
import pytest

import oracle as O
from parity_util import MAX_TOL, RMS_TOL, compare_x, gpu_opts, oracle_opts
from workloads import make

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1511_03296_b200 as fbs


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run_gpu(w, n_irls, **over):
    g = fbs.grid_build(dev(w.rgb), w.sigma_xy, w.sigma_l, w.sigma_uv, n_bistoch=w.n_bistoch)
    x, c = fbs.solve_robust(g, dev(w.t), dev(w.c), w.lam, w.sigma_gm, n_irls, want_weights=True,
                            **gpu_opts(w, **over))
    torch.cuda.synchronize()
    return g, x.cpu().numpy(), c.cpu().numpy()


@pytest.mark.parametrize("variant", ["hier_fixed", "jacobi_tol"])
def test_robust_parity(variant):
    """Both sides run Alg. 3 with the same inner solver settings; x̂ within north_star's bounds."""
    w = make("rbs", W=203, H=151, n_cells=30, n_irls=4)
    over = {} if variant == "hier_fixed" else dict(precond="jacobi", init="flat", mode="tol", tol=1e-6)
    g, x, c = run_gpu(w, w.n_irls, **over)
    _, out = O.robust_solve(w.rgb, w.t, w.c, w.sigma_xy, w.sigma_l, w.sigma_uv, w.lam, oracle_opts(w, **over),
                            w.sigma_gm, w.n_irls)
    HW = w.H * w.W
    mx, rms = compare_x(x[0].reshape(1, HW), out[0].sol.x, w.t[0].reshape(1, HW).astype(float),
                        np.ones(HW))
    assert mx <= MAX_TOL and rms <= RMS_TOL, (mx, rms)
    # the final weights are a smooth function of x̂: relative agreement on the same scale
    wr = out[0].weights
    assert np.abs(c[0].ravel() - wr).max() <= 1e-2 * wr.max()


def test_one_round_equals_plain_solve():
    w = make("rbs", W=128, H=96, n_cells=20, n_irls=1)
    g = fbs.grid_build(dev(w.rgb), w.sigma_xy, w.sigma_l, w.sigma_uv)
    t, c = dev(w.t), dev(w.c)
    x1 = fbs.solve_robust(g, t, c, w.lam, w.sigma_gm, 1, **gpu_opts(w))
    x2 = fbs.solve(g, t, c, w.lam, **gpu_opts(w))
    torch.cuda.synchronize()
    assert torch.equal(x1, x2)


def test_argument_errors():
    w = make("rbs", W=64, H=48, n_cells=8)
    g = fbs.grid_build(dev(w.rgb), w.sigma_xy, w.sigma_l, w.sigma_uv)
    t, c = dev(w.t), dev(w.c)
    with pytest.raises(fbs.FbsError):
        fbs.solve_robust(g, t, c, w.lam, 0.0, 2)
    with pytest.raises(fbs.FbsError):
        fbs.solve_robust(g, t, c, w.lam, 5.0, 0)
    with pytest.raises(fbs.FbsError):
        fbs.solve_robust(g, t.repeat(1, 2, 1, 1), c, w.lam, 5.0, 2)


def test_robust_rejects_outliers_at_scale():
    """640×480, 10% unflagged outliers, 8 IRLS rounds: closer to the clean depth than the plain
    solver (the oracle pin test_rbs_rejects_unflagged_outliers, here on the CUDA path)."""
    w = make("rbs")
    g, x, _ = run_gpu(w, w.n_irls)
    xp = fbs.solve(g, dev(w.t), dev(w.c), w.lam, **gpu_opts(w)).cpu().numpy()
    truth = w.truth[0]
    mae_r = np.abs(x[0, 0] - truth).mean()
    mae_p = np.abs(xp[0, 0] - truth).mean()
    assert mae_r < 0.3 * mae_p, (mae_r, mae_p)
