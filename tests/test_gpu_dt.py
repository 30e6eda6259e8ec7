"""GPU parity of the domain-transform post-filter (fbs_dt_filter) against the oracle's
recursion (reading #28), including ragged line lengths (not multiples of 32, shorter than 32)."""
import numpy as np
import pytest

import oracle as O
from workloads import make

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1511_03296_b200 as fbs


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


# tall planes (H = 1536, 1600): long column recursions across many warp chunks; H = 1080, 1152:
# the register-resident column kernel (up to its 64 × 18 rows), 1153: the transpose path;
# W = 260, 1028, 1920: rows of ≥ 256 pixels take two warps per row (k_dt_rows2)
@pytest.mark.parametrize("H,W,K,ss,sr", [(48, 64, 1, 16.0, 16.0), (37, 203, 2, 4.0, 8.0), (5, 17, 1, 8.0, 4.0),
                                         (130, 9, 3, 32.0, 64.0), (1, 77, 1, 4.0, 4.0), (1600, 40, 1, 16.0, 8.0),
                                         (1536, 33, 1, 8.0, 16.0), (1152, 48, 1, 16.0, 16.0), (1080, 100, 2, 16.0, 8.0),
                                         (1153, 20, 1, 16.0, 16.0), (40, 1920, 1, 16.0, 16.0), (33, 260, 2, 8.0, 4.0),
                                         (7, 1028, 1, 32.0, 8.0)])
def test_dt_parity(H, W, K, ss, sr):
    w = make("c2", W=W, H=H, n_cells=6)
    rng = np.random.default_rng(H * 1000 + W)
    x = (rng.normal(size=(2, K, H, W)) * 40 + 100).astype(np.float32)
    rgb = np.concatenate([w.rgb, w.rgb[:, ::-1].copy()])
    y = fbs.dt_filter(dev(rgb), dev(x), ss, sr).cpu().numpy()
    for f in range(2):
        ref = O.dt_filter(x[f].astype(np.float64), rgb[f], ss, sr)
        rngv = float(x[f].max() - x[f].min())
        d = np.abs(y[f] - ref)
        assert d.max() <= 1e-4 * rngv and np.sqrt(np.mean(d * d)) <= 1e-5 * rngv, (d.max() / rngv)


def test_dt_in_place_and_constant():
    w = make("c1")
    x = np.full((1, 2, w.H, w.W), 3.5, np.float32)
    xt = dev(x)
    fbs.dt_filter(dev(w.rgb), xt, 16.0, 16.0, out=xt)
    torch.cuda.synchronize()
    assert torch.allclose(xt, torch.full_like(xt, 3.5), rtol=1e-6)


def test_solve_then_dt_pipeline():
    """The paper's pipeline: solve, then post-filter with σ'_xy = σ'_rgb = 16."""
    w = make("c2", W=160, H=120, n_cells=20)
    g = fbs.grid_build(dev(w.rgb), w.sigma_xy, w.sigma_l, w.sigma_uv)
    x = fbs.solve(g, dev(w.t), dev(w.c), w.lam, precond="hier", init="hier", mode="fixed", iters=25)
    y = fbs.dt_filter(dev(w.rgb), x, 16.0, 16.0).cpu().numpy()
    ref = O.dt_filter(x.cpu().numpy()[0].astype(np.float64), w.rgb[0], 16.0, 16.0)
    assert np.abs(y[0] - ref).max() <= 1e-4 * float(w.t.max() - w.t.min())
