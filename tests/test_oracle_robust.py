"""Oracle pins for the robust bilateral solver (Supp. §3, Alg. 3).

Each test checks oracle.robust_solve against something other than its own formula: a
derivative identity, a brute-force scalar IRLS written independently, the plain solver the
algorithm must reduce to, an invariant, or the majorize–minimize property (reading #25).
"""
import numpy as np
import pytest

import oracle as O
from workloads import make


def test_gm_weight_is_rho_prime_over_e():
    """IRLS weight consistency (Supp. §3): w(e) = ρ'(e)/e, with ρ' by central differences."""
    for sg in (0.5, 1.0, 7.0):
        e = np.linspace(-40, 40, 161)
        e = e[np.abs(e) > 1e-3]
        h = 1e-6 * np.maximum(1.0, np.abs(e))
        d = (O.gm_rho(e + h, sg) - O.gm_rho(e - h, sg)) / (2 * h)
        np.testing.assert_allclose(O.gm_weight(e, sg), d / e, rtol=1e-6, atol=1e-12)
    # asymptotes: ρ(0) = 0, ρ → 1 and w → 0 as |e| → ∞ ("a smooth approximation to the ℓ0-norm")
    assert O.gm_rho(0.0, 2.0) == 0.0 and abs(O.gm_rho(1e9, 2.0) - 1.0) < 1e-12 and O.gm_weight(1e9, 2.0) < 1e-30


def _one_vertex_image(t_vals):
    """A constant-colour image whose pixels all fall in one σxy cell: a one-vertex grid, where
    the solver reduces to the confidence-weighted mean (A = S c, b = S(c∘t))."""
    n = len(t_vals)
    W = 4
    H = (n + W - 1) // W
    assert H * W == n
    rgb = np.full((1, H, W, 3), 120, np.uint8)
    t = np.asarray(t_vals, np.float64).reshape(1, 1, H, W)
    return rgb, t


def test_scalar_irls_matches_bruteforce():
    """One vertex: x̂ = Σ c t / Σ c each round, so Alg. 3 is the scalar IRLS below."""
    rng = np.random.default_rng(7)
    t_vals = np.concatenate([rng.normal(10.0, 0.3, 14), [60.0, -45.0]])
    rgb, t = _one_vertex_image(t_vals)
    c0 = rng.uniform(0.5, 1.5, t_vals.size)
    sg, n = 1.5, 12
    grid, out = O.robust_solve(rgb, t, c0.reshape(1, *t.shape[2:]), 8.0, 8.0, 8.0, 3.0,
                               O.SolveOptions(mode="tol", tol=1e-14), sg, n)
    assert grid.M == 1
    # independent scalar IRLS
    c = c0.copy()
    for _ in range(n):
        x = np.sum(c * t_vals) / np.sum(c)
        c = 2 * sg * sg / (sg * sg + (x - t_vals) ** 2) ** 2
    np.testing.assert_allclose(out[0].sol.x[0], x, rtol=1e-12)
    np.testing.assert_allclose(out[0].weights, c, rtol=1e-10)
    # the outliers are rejected: x̂ near the inlier mean, outlier weights < 1% of inlier weights
    assert abs(x - np.mean(t_vals[:14])) < 0.3
    assert c[14:].max() < 0.01 * c[:14].min()


def test_large_sigma_reduces_to_plain_solver():
    """σ_gm → ∞: w → 2/σ² everywhere, and (c, λ) → (κc, κλ) leaves the solution unchanged
    (reading #16), so rounds ≥ 2 equal the plain solver with c = 1 and λ' = λσ²/2."""
    w = make("c2", W=48, H=40)
    H, W = w.H, w.W
    opts = O.SolveOptions(mode="tol", tol=1e-13, max_iters=20000)
    sg = 1e5
    grid, out = O.robust_solve(w.rgb, w.t, w.c, w.sigma_xy, w.sigma_l, w.sigma_uv, w.lam, opts, sg, 3)
    plain = O.solve_frame(grid, 0, w.t[0].reshape(1, H * W).astype(float), np.ones(H * W), w.lam * sg * sg / 2,
                          opts)
    rng_t = float(w.t.max() - w.t.min())
    # w = (2/σ²)(1 + e²/σ²)⁻²: the rounds differ from the plain solve by O(e²/σ²) ≤ 7e-6 here;
    # a wrong factor in w (e.g. σ² instead of 2σ²) would double λ' and miss by percents
    assert np.abs(out[0].sol.x[0] - plain.x[0]).max() < 1e-4 * rng_t


def test_constant_target_fixed_point():
    """A constant target is reproduced exactly at every round, with weights 2/σ²."""
    w = make("c1")
    t = np.full_like(w.t, 3.25)
    grid, out = O.robust_solve(w.rgb, t, w.c, w.sigma_xy, w.sigma_l, w.sigma_uv, w.lam,
                               O.SolveOptions(mode="tol", tol=1e-13), 2.0, 3)
    np.testing.assert_allclose(out[0].sol.x[0], 3.25, atol=1e-8)
    np.testing.assert_allclose(out[0].weights, 2 / 4.0, rtol=1e-8)


def test_one_round_is_the_plain_solve():
    w = make("c1")
    HW = w.H * w.W
    opts = O.SolveOptions(mode="tol", tol=1e-10)
    grid, out = O.robust_solve(w.rgb, w.t, w.c, w.sigma_xy, w.sigma_l, w.sigma_uv, w.lam, opts, 0.2, 1)
    _, sols = O.solve(w.rgb, w.t, w.c, w.sigma_xy, w.sigma_l, w.sigma_uv, w.lam, opts)
    np.testing.assert_array_equal(out[0].sol.x, sols[0].x)
    np.testing.assert_allclose(out[0].weights, O.gm_weight(sols[0].x[0] - w.t[0].reshape(HW), 0.2))


def test_mm_objective_non_increasing():
    """Reading #25: c ← w(e) makes each exact inner solve minimise a majoriser of
    λ/2 Σ Ŵ (x_i − x_j)² + 2 Σ ρ(e_i) (ρ is concave in e²), so that objective never increases."""
    w = make("rbs", W=80, H=64, n_irls=6)
    opts = O.SolveOptions(mode="tol", tol=1e-12, max_iters=20000)
    _, out = O.robust_solve(w.rgb, w.t, w.c, w.sigma_xy, w.sigma_l, w.sigma_uv, w.lam, opts, w.sigma_gm,
                            w.n_irls)
    mm = out[0].mm_losses
    assert all(b <= a * (1 + 1e-9) for a, b in zip(mm, mm[1:])), mm


def test_rbs_rejects_unflagged_outliers():
    """Robustness: with 10% uniform outliers that c_init does not flag, the
    RBS output is closer to the clean depth than the plain solver's."""
    w = make("rbs", W=120, H=96, n_irls=8)
    opts = O.SolveOptions(precond="hier", init="hier", mode="fixed", iters=25)
    grid, out = O.robust_solve(w.rgb, w.t, w.c, w.sigma_xy, w.sigma_l, w.sigma_uv, w.lam, opts, w.sigma_gm,
                               w.n_irls)
    _, plain = O.solve(w.rgb, w.t, w.c, w.sigma_xy, w.sigma_l, w.sigma_uv, w.lam, opts)
    truth = w.truth[0].ravel()
    mae_rbs = np.abs(out[0].sol.x[0] - truth).mean()
    mae_plain = np.abs(plain[0].x[0] - truth).mean()
    assert mae_rbs < 0.7 * mae_plain, (mae_rbs, mae_plain)
