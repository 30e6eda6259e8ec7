"""Oracle pins for the domain-transform post-filter (reading #28)."""
import numpy as np
import pytest
import scipy.linalg as sla

import oracle as O
from workloads import make


def test_constant_signal_unchanged_and_linear():
    w = make("c1")
    rgb = w.rgb[0]
    H, W = w.H, w.W
    out = O.dt_filter(np.full((1, H, W), 7.5), rgb, 16.0, 16.0)
    np.testing.assert_allclose(out, 7.5, rtol=1e-13)
    rng = np.random.default_rng(0)
    a, b = rng.normal(size=(2, 1, H, W))
    np.testing.assert_allclose(O.dt_filter(2 * a - 3 * b, rgb, 8.0, 20.0),
                               2 * O.dt_filter(a, rgb, 8.0, 20.0) - 3 * O.dt_filter(b, rgb, 8.0, 20.0), atol=1e-10)


def _dense_pass(f, V):
    """One causal + anticausal pass along a 1-D line as two dense triangular solves:
    causal (I − diag(w) L) J = diag(1 − w) f with w_0 = 0; anticausal likewise reversed."""
    n = f.size
    w = V.copy()
    w[0] = 0.0
    L = np.diag(-w[1:], -1) + np.eye(n)
    J = sla.solve_triangular(L, (1 - w) * f, lower=True)
    u = np.append(V[1:], 0.0)  # element k uses w[k+1]
    U = np.diag(-u[:-1], 1) + np.eye(n)
    return sla.solve_triangular(U, (1 - u) * J, lower=False)


def test_rows_and_columns_equal_dense_triangular_solves():
    """The recursion of each pass equals its lower/upper bidiagonal linear systems (independent
    route through LAPACK triangular solves), pass by pass and line by line."""
    rng = np.random.default_rng(1)
    H, W = 7, 9
    rgb = rng.integers(0, 256, (H, W, 3)).astype(np.uint8)
    f = rng.normal(size=(1, H, W))
    ss, sr = 6.0, 30.0
    I = rgb.astype(float)
    Dx = np.ones((H, W))
    Dx[:, 1:] += ss / sr * np.abs(np.diff(I, axis=1)).sum(axis=2)
    Dy = np.ones((H, W))
    Dy[1:, :] += ss / sr * np.abs(np.diff(I, axis=0)).sum(axis=2)
    ref = f[0].copy()
    N = 2
    for i in (1, 2):
        a = np.exp(-np.sqrt(2) / (ss * np.sqrt(3) * 2 ** (N - i) / np.sqrt(4 ** N - 1)))
        ref = np.stack([_dense_pass(ref[y], a ** Dx[y]) for y in range(H)])
        ref = np.stack([_dense_pass(ref[:, x], a ** Dy[:, x]) for x in range(W)], axis=1)
    np.testing.assert_allclose(O.dt_filter(f, rgb, ss, sr, n_iters=N)[0], ref, rtol=1e-12, atol=1e-12)


def test_edge_preserving():
    """A guide step of 255 with σ_r small: a signal step aligned with it survives (away from
    the edge the output stays within 1% of the step height)."""
    H, W = 24, 64
    rgb = np.zeros((H, W, 3), np.uint8)
    rgb[:, W // 2:] = 255
    f = np.zeros((1, H, W))
    f[:, :, W // 2:] = 100.0
    out = O.dt_filter(f, rgb, 8.0, 4.0)
    assert np.abs(out[0, :, : W // 2 - 3]).max() < 1.0
    assert np.abs(out[0, :, W // 2 + 3:] - 100.0).max() < 1.0
    # and without the guide edge the step is smoothed out
    flat = O.dt_filter(f, np.zeros_like(rgb), 8.0, 4.0)
    assert abs(flat[0, H // 2, W // 2 - 2] - 50.0) < 30.0 and flat[0, H // 2, W // 2 - 2] > 5.0


def test_sigma_schedule_sums_to_sigma_s():
    """The schedule's defining property (Gastal & Oliveira 2011, reading #28): the N passes'
    variances add up to the requested σ_s² (Σ σ_i² = σ_s²), each pass halves the previous
    pass's σ (the widest kernel first)."""
    for ss, N in ((8.0, 3), (30.0, 3), (5.0, 1), (12.0, 5)):
        sig = O.dt_sigmas(ss, N)
        assert len(sig) == N
        assert np.sum(sig ** 2) == pytest.approx(ss * ss, rel=1e-12)
        assert np.allclose(sig[:-1] / sig[1:], 2.0, rtol=1e-12)


def test_impulse_response_variance_on_flat_guide():
    """Behavioural pin of the whole filter on a flat guide (d ≡ 1): each pass's causal +
    anticausal recursion has an impulse response of variance 2a/(1−a)² ≈ σ_i² (a = e^{−√2/σ_i}),
    so the filtered impulse keeps unit mass and its variance along x is ≈ σ_s² (within 1.5 % for
    σ_s ≥ 8) — a wrong normalisation or base of the schedule fails."""
    W = 1601
    for ss in (8.0, 30.0):
        f = np.zeros((1, 1, W))
        f[0, 0, W // 2] = 1.0
        out = O.dt_filter(f, np.zeros((1, W, 3), np.uint8), ss, 10.0)[0, 0]
        xs = np.arange(W) - W // 2
        assert out.sum() == pytest.approx(1.0, abs=1e-9)
        var = float(np.sum(out * xs * xs))
        assert var == pytest.approx(ss * ss, rel=0.015)
