"""Oracle pins for the low-rank multi-RHS reduction (Supp. §4).

reduce_rhs is checked against hand-computable cases and the Frobenius bound its tolerance
promises; the reduced solve against the full per-channel solve it approximates (exactly, for
ε = 0 and exact inner solves)."""
import numpy as np

import oracle as O
from workloads import make


def test_duplicate_columns_rank_one():
    rng = np.random.default_rng(1)
    b = rng.normal(size=500)
    B = np.stack([b, b, 2 * b], axis=1)
    red = O.reduce_rhs(B, 0.01)
    assert red.t == 1
    np.testing.assert_allclose(red.Q @ red.R, B, atol=1e-12 * np.abs(B).max())


def test_orthogonal_masses_example():
    """Orthogonal columns with masses [100, 1, 1e-4], ε = 0.01: the first row alone keeps
    100/101.0001 ≥ 0.99 of the mass → t = 1 (hand computation)."""
    M = 300
    B = np.zeros((M, 3))
    B[0, 0], B[1, 1], B[2, 2] = 10.0, 1.0, 1e-2
    red = O.reduce_rhs(B, 0.01)
    assert red.t == 1
    np.testing.assert_allclose(red.masses, [100.0, 1.0, 1e-4], rtol=1e-12)
    assert O.reduce_rhs(B, 0.001).t == 2 and O.reduce_rhs(B, 0.0).t == 3


def test_frobenius_bound_orthonormal_and_monotone():
    rng = np.random.default_rng(2)
    U = rng.normal(size=(2000, 4))
    B = U @ rng.normal(size=(4, 21)) + 1e-3 * rng.normal(size=(2000, 21))
    prev = 22
    for eps in (0.0, 1e-6, 1e-3, 0.01, 0.1, 0.5):
        red = O.reduce_rhs(B, eps)
        assert red.t <= prev
        prev = red.t
        np.testing.assert_allclose(red.Q.T @ red.Q, np.eye(red.t), atol=1e-10)
        resid = np.sum((B - red.Q @ red.R) ** 2)
        assert resid <= eps * np.sum(B * B) + 1e-9 * np.sum(B * B), (eps, resid)
    assert O.reduce_rhs(B, 0.01).t == 4


def test_eps_zero_equals_per_channel_solve():
    w = make("c4", W=60, H=45, n_cells=6, K=5)
    opts = O.SolveOptions(precond="jacobi", init="flat", mode="tol", tol=1e-12, max_iters=20000)
    grid = O.build_grid(w.rgb, w.sigma_xy, w.sigma_l, w.sigma_uv)
    HW = w.H * w.W
    t = w.t[0].reshape(5, HW).astype(float)
    c = w.c[0].reshape(HW).astype(float)
    x_lr, Y, red = O.solve_frame_lowrank(grid, 0, t, c, w.lam, opts, 0.0)
    full = O.solve_frame(grid, 0, t, c, w.lam, opts)
    assert red.t == 5
    np.testing.assert_allclose(x_lr, full.x, atol=1e-8)


def test_rank4_reduced_solve_close_to_full():
    """21 channels of effective rank 4 (+1e-6 noise), ε = 0.01: t ≤ 5 and the expanded solution
    within 1e-3 of each channel's range of the full per-channel solve."""
    w = make("c4", W=80, H=60, n_cells=10)
    HW = w.H * w.W
    rng = np.random.default_rng(3)
    base = w.t[0, :4].reshape(4, HW).astype(float)
    t = rng.normal(size=(21, 4)) @ base + 1e-6 * rng.normal(size=(21, HW))
    c = w.c[0].reshape(HW).astype(float)
    opts = O.SolveOptions(precond="hier", init="hier", mode="tol", tol=1e-10, max_iters=20000)
    grid = O.build_grid(w.rgb, w.sigma_xy, w.sigma_l, w.sigma_uv)
    x_lr, _, red = O.solve_frame_lowrank(grid, 0, t, c, w.lam, opts, 0.01)
    full = O.solve_frame(grid, 0, t, c, w.lam, opts)
    assert red.t <= 5
    rng_k = t.max(axis=1) - t.min(axis=1)
    assert np.all(np.abs(x_lr - full.x).max(axis=1) <= 1e-3 * rng_k)
