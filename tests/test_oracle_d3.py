"""Oracle pins for the grayscale (D = 3, XYL) grid (PAPER.md:511 colorization; reading #27)."""
import numpy as np
import scipy.linalg as sla

import oracle as O
from workloads import make


def gray(vals, H, W):
    v = np.asarray(vals, np.uint8).reshape(1, H, W, 1)
    return np.repeat(v, 3, axis=3)


def test_1x2_gray_examples():
    """identical gray pixels coalesce; 0 and 255 at σl = 8 land in luma cells
    ⌊0/8⌋ = 0 and ⌊255/8⌋ = 31, which are not adjacent (hand quantisation)."""
    g = O.build_grid(gray([128, 128], 1, 2), 16.0, 8.0, 8.0, dims=3)
    assert g.M == 1 and list(g.m) == [2]
    g = O.build_grid(gray([0, 255], 1, 2), 16.0, 8.0, 8.0, dims=3)
    assert g.M == 2 and list(g.m) == [1, 1]
    assert sorted(g.V[:, O.COL["l"]].tolist()) == [0, 31]
    assert np.all(g.nbr == -1)


def test_gray_image_same_structure_as_d5():
    """A gray reference has constant chroma, so its 5-D grid has the 3-D grid's vertices,
    splat map and links — only the constant chroma coordinates differ."""
    rng = np.random.default_rng(4)
    img = gray(rng.integers(0, 256, 40 * 56), 40, 56)
    g5 = O.build_grid(img, 8.0, 4.0, 3.0, dims=5)
    g3 = O.build_grid(img, 8.0, 4.0, 3.0, dims=3)
    assert np.array_equal(g5.vid, g3.vid) and np.array_equal(g5.m, g3.m) and np.array_equal(g5.nbr, g3.nbr)
    assert np.all(g3.V[:, O.COL["u"]] == 0) and np.all(g3.V[:, O.COL["v"]] == 0)


def test_d3_blur_and_bistoch_closed_forms():
    """B̄ = 6I + Adj (reading #4 with D = 3): [1] → [6]; Alg. 1 gives n = √(m/6) for an isolated
    vertex and √(m/7) for a symmetric adjacent pair."""
    B = O.blur_matrix(np.full((1, 10), -1), dims=3)
    assert B.toarray().tolist() == [[6.0]]
    n, _ = O.bistochastize(np.array([5]), B, 20)
    np.testing.assert_allclose(n, np.sqrt(5 / 6), rtol=1e-14)
    nbr = np.full((2, 10), -1)
    nbr[0, 1], nbr[1, 0] = 1, 0
    n, _ = O.bistochastize(np.array([4, 4]), O.blur_matrix(nbr, dims=3), 40)
    np.testing.assert_allclose(n, np.sqrt(4 / 7), rtol=1e-12)


def test_d3_solve_matches_cholesky():
    """A colorization-style problem on a gray reference (sparse confidence): PCG to 1e-12
    equals the dense Cholesky solve of the same A (A SPD)."""
    w = make("c1")
    img = np.repeat(w.rgb[..., :1], 3, axis=3)
    c = np.where(np.random.default_rng(5).uniform(size=w.c.shape) < 0.2, 1.0, 0.0).astype(np.float32)
    c[..., 0, 0] = 1.0
    _, sols = O.solve(img, w.t, c, 8.0, 8.0, 8.0, 4.0, O.SolveOptions(mode="tol", tol=1e-13, max_iters=10000),
                      dims=3)
    s = sols[0]
    A = s.sys.A.toarray()
    live = s.sys.live
    comp = O.zero_confidence_components(s.nbr, s.sys.Sc)
    keep = live & ~comp
    Ak = A[np.ix_(keep, keep)]
    assert np.all(np.linalg.eigvalsh(0.5 * (Ak + Ak.T)) > 0)
    y = sla.cho_solve(sla.cho_factor(Ak), s.sys.b[keep, 0])
    np.testing.assert_allclose(s.y[keep, 0], y, rtol=1e-8, atol=1e-9 * np.abs(y).max())
