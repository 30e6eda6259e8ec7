"""GPU parity of the low-rank multi-RHS solve (Supp. §4, opts.lowrank_eps) against the oracle's
reduce_rhs + reduced solve, and its consistency with the full per-channel solve."""
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


@pytest.mark.parametrize("variant", ["jacobi_tol", "hier_fixed"])
def test_lowrank_parity(variant):
    """configs[3]-like 21-channel class probabilities, ε = 0.01: same reduction, same solves."""
    w = make("c4", W=150, H=112, n_cells=12)
    over = {} if variant == "jacobi_tol" else dict(precond="hier", init="hier", mode="fixed", iters=25)
    g = fbs.grid_build(dev(w.rgb), w.sigma_xy, w.sigma_l, w.sigma_uv)
    x = fbs.solve(g, dev(w.t), dev(w.c), w.lam, lowrank_eps=0.01, **gpu_opts(w, **over)).cpu().numpy()
    grid = O.build_grid(w.rgb, w.sigma_xy, w.sigma_l, w.sigma_uv)
    HW = w.H * w.W
    t = w.t[0].reshape(w.t.shape[1], HW).astype(float)
    c = w.c[0].reshape(HW).astype(float)
    x_ref, _, red = O.solve_frame_lowrank(grid, 0, t, c, w.lam, oracle_opts(w, **over), 0.01)
    assert red.t < t.shape[0]
    mx, rms = compare_x(x[0].reshape(t.shape[0], HW), x_ref, t, c)
    assert mx <= MAX_TOL and rms <= RMS_TOL, (mx, rms, red.t)


def test_tiny_eps_matches_full_solve():
    """ε → 0 keeps every row: Y = A⁻¹ Q R = A⁻¹ B, the per-channel solve (both to tol 1e-6)."""
    w = make("c4", W=120, H=90, n_cells=10, K=6)
    g = fbs.grid_build(dev(w.rgb), w.sigma_xy, w.sigma_l, w.sigma_uv)
    t, c = dev(w.t), dev(w.c)
    x_lr = fbs.solve(g, t, c, w.lam, lowrank_eps=1e-12, **gpu_opts(w)).cpu().numpy()
    x_full = fbs.solve(g, t, c, w.lam, **gpu_opts(w)).cpu().numpy()
    HW = w.H * w.W
    mx, rms = compare_x(x_lr[0].reshape(6, HW), x_full[0].reshape(6, HW).astype(float),
                        w.t[0].reshape(6, HW).astype(float), w.c[0].reshape(HW))
    assert mx <= MAX_TOL and rms <= RMS_TOL, (mx, rms)


def test_lowrank_batch_frames_independent():
    """Each frame is reduced on its own (its own t_f): a frame solved in a batch equals the same
    frame solved alone."""
    w = make("c4", W=96, H=72, n_cells=8, K=8)
    rgb2 = np.concatenate([w.rgb, w.rgb[:, ::-1].copy()])
    t2 = np.concatenate([w.t, w.t[:, :, ::-1] * 0.5])
    c2 = np.concatenate([w.c, w.c[:, ::-1]])
    gb = fbs.grid_build(dev(rgb2), w.sigma_xy, w.sigma_l, w.sigma_uv)
    xb = fbs.solve(gb, dev(t2), dev(c2), w.lam, lowrank_eps=0.01, **gpu_opts(w)).cpu().numpy()
    g1 = fbs.grid_build(dev(w.rgb), w.sigma_xy, w.sigma_l, w.sigma_uv)
    x1 = fbs.solve(g1, dev(w.t), dev(w.c), w.lam, lowrank_eps=0.01, **gpu_opts(w)).cpu().numpy()
    rng = float(w.t.max() - w.t.min())
    assert np.abs(xb[0] - x1[0]).max() <= 1e-4 * rng


def test_lowrank_rejects_keep_system():
    w = make("c4", W=64, H=48, n_cells=6, K=4)
    g = fbs.grid_build(dev(w.rgb), w.sigma_xy, w.sigma_l, w.sigma_uv)
    with pytest.raises(fbs.FbsError):
        fbs.solve(g, dev(w.t), dev(w.c), w.lam, keep_system=True, lowrank_eps=0.01, **gpu_opts(w))
    with pytest.raises(fbs.FbsError):
        fbs.solve(g, dev(w.t), dev(w.c), w.lam, lowrank_eps=1.5, **gpu_opts(w))
