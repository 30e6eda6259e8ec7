"""Pins for the fp64 oracle (CPU only).

Each test checks the oracle against something other than itself: worked examples
(tests/golden/, with citations), closed forms, brute force on tiny inputs, dense
LAPACK solves, finite differences and invariants the paper states.  Chosen so that a
dropped term, a wrong sign/index or a transposed operand in oracle/ fails one of them.
"""

import numpy as np
import pytest
import scipy.linalg as sla

import oracle as O
from workloads import make


def const_image(rgb, H, W, F=1):
    return np.broadcast_to(np.array(rgb, np.uint8), (F, H, W, 3)).copy()


def frame_solve(rgb, t, c, sxy, sl, suv, lam, **kw):
    opts = O.SolveOptions(**kw)
    grid = O.build_grid(rgb, sxy, sl, suv)
    t = np.asarray(t, np.float64).reshape(-1, rgb.shape[1] * rgb.shape[2])
    c = np.asarray(c, np.float64).reshape(-1)
    return grid, O.solve_frame(grid, 0, t, c, lam, opts)


def tiny_case(seed=7, W=24, H=18, K=1, sxy=4.0, sl=16.0, suv=16.0, cells=5):
    rng = np.random.default_rng(seed)
    from workloads.synth import voronoi_reference
    rgb, lab, _ = voronoi_reference(rng, W, H, cells, "gradient", 6.0)
    t = rng.uniform(0, 1, (K, H * W))
    c = rng.uniform(0.2, 1.0, H * W)
    return rgb[None], t, c, sxy, sl, suv


# ----------------------------------------------------------------------------- grid
def test_gray_yuv(worked):
    for k, yn, un, vn in worked["gray_yuv"]["cases"]:
        Y, U, V = O.yuv_numerators(np.array([[k, k, k]], np.uint8))
        assert (int(Y[0]), int(U[0]), int(V[0])) == (yn, un, vn)
    k = np.arange(256, dtype=np.uint8)
    Y, U, V = O.yuv_numerators(np.stack([k, k, k], 1))
    assert np.array_equal(Y, 256 * k.astype(np.int64)) and np.all(U == 32768) and np.all(V == 32768)


def test_bt601_primaries(worked):
    """Reading #1 pinned on the channel order: the numerators of pure R, G and B (golden, derived
    from BT.601's Kr, Kb), and on random colours the oracle's (l, u − 128, v − 128) agree with
    BT.601 evaluated from its defining constants (Y = Kr R + (1−Kr−Kb) G + Kb B,
    U = (B − Y)/(2(1 − Kb)), V = (R − Y)/(2(1 − Kr))) to within the 8-bit coefficient rounding
    (≤ ½/256 per coefficient, × 3 × 255).  An RGB↔BGR swap or a U↔V swap fails both."""
    ex = worked["bt601_primaries"]
    for rgb, nums in ex["cases"]:
        Y, U, V = O.yuv_numerators(np.array([rgb], np.uint8))
        assert (int(Y[0]), int(U[0]), int(V[0])) == tuple(nums)
    kr, kb = ex["Kr"], ex["Kb"]
    px = np.random.default_rng(11).integers(0, 256, (4096, 3)).astype(np.uint8)
    R, G, B = (px[:, i].astype(np.float64) for i in range(3))
    Yr = kr * R + (1 - kr - kb) * G + kb * B
    Ur = (B - Yr) / (2 * (1 - kb))
    Vr = (R - Yr) / (2 * (1 - kr))
    Y, U, V = O.yuv_numerators(px)
    bound = 3 * 255 * 0.5 / 256
    assert np.abs(Y / 256 - Yr).max() <= bound
    assert np.abs(U / 256 - 128 - Ur).max() <= bound
    assert np.abs(V / 256 - 128 - Vr).max() <= bound


@pytest.mark.parametrize("sxy,num,den", [(8.0, 1, 8), (7.5, 2, 15), (3.0, 1, 3), (1.0, 1, 1)])
@pytest.mark.parametrize("sl,suv", [(8.0, 8.0), (4.0, 3.0), (4.0, 4.0), (1.0, 1.0)])
def test_bins_equal_integer_floor(sxy, num, den, sl, suv):
    """Reading #2: floor of an fp64 division equals exact integer floor division here
    (independent integer computation: sxy = den/num, 256·σ integer)."""
    rng = np.random.default_rng(3)
    rgb = rng.integers(0, 256, (2, 13, 17, 3), dtype=np.uint8)
    P = O.pixel_coords(rgb, sxy, sl, suv)
    F, H, W, _ = rgb.shape
    r, g, b = (rgb[..., i].astype(np.int64).ravel() for i in range(3))
    ys = np.repeat(np.tile(np.arange(H), F), W)
    xs = np.tile(np.arange(W), F * H)
    assert np.array_equal(P[:, 1], (ys * num) // den)
    assert np.array_equal(P[:, 2], (xs * num) // den)
    assert np.array_equal(P[:, 3], (77 * r + 150 * g + 29 * b) // int(256 * sl))
    assert np.array_equal(P[:, 4], (-43 * r - 85 * g + 128 * b + 32768) // int(256 * suv))
    assert np.array_equal(P[:, 5], (128 * r - 107 * g - 21 * b + 32768) // int(256 * suv))


def test_grid_4x4_constant(worked):
    ex = worked["grid_4x4_constant"]
    g = O.build_grid(const_image(ex["rgb"], ex["H"], ex["W"]), ex["sigma_xy"], ex["sigma_l"], ex["sigma_uv"])
    assert g.M == ex["M"]
    assert list(g.m) == ex["m"]
    assert list(g.vid) == ex["vid"]
    assert g.nbr[:, 0:2].tolist() == ex["nbr_x"]
    assert g.nbr[:, 2:4].tolist() == ex["nbr_y"]
    assert np.all(g.nbr[:, 4:] == -1)


def test_grid_1x2_coalesce(worked):
    ex = worked["grid_1x2_coalesce"]
    g = O.build_grid(const_image(ex["rgb"], ex["H"], ex["W"]), ex["sigma_xy"], ex["sigma_l"], ex["sigma_uv"])
    assert g.M == ex["M"] and list(g.m) == ex["m"]


def _int_tuples(rgb, num, den, sl, suv):
    F, H, W, _ = rgb.shape
    r, g, b = (rgb[..., i].astype(np.int64).ravel() for i in range(3))
    fr = np.repeat(np.arange(F), H * W)
    ys = np.repeat(np.tile(np.arange(H), F), W)
    xs = np.tile(np.arange(W), F * H)
    return np.stack([fr, (ys * num) // den, (xs * num) // den, (77 * r + 150 * g + 29 * b) // int(256 * sl),
                     (-43 * r - 85 * g + 128 * b + 32768) // int(256 * suv),
                     (128 * r - 107 * g - 21 * b + 32768) // int(256 * suv)], 1)


@pytest.mark.parametrize("frames", [1, 2])
def test_grid_bruteforce(frames):
    """O(N²) brute force: same vid ⇔ same integer tuple; m counts; keys ascending; O(M²) neighbours."""
    w = make("c1")
    rgb = np.concatenate([w.rgb] * frames)
    if frames == 2:
        rgb[1] = np.flip(rgb[1], axis=1)
    g = O.build_grid(rgb, 8.0, 8.0, 8.0)
    T = _int_tuples(rgb, 1, 8, 8.0, 8.0)
    same_tuple = np.all(T[:, None, :] == T[None, :, :], axis=2)
    same_vid = g.vid[:, None] == g.vid[None, :]
    assert np.array_equal(same_tuple, same_vid)
    assert np.array_equal(g.V[g.vid], T)
    assert np.array_equal(np.bincount(g.vid, minlength=g.M), g.m) and g.m.sum() == rgb[..., 0].size
    keys = g.keys
    assert np.all(keys[1:] > keys[:-1])
    # neighbours: u is the ±e_d neighbour of v ⇔ tuples differ by exactly ±1 in dim d only
    col = [2, 1, 3, 4, 5]
    diff = g.V[None, :, :] - g.V[:, None, :]  # [v][u] = V[u] - V[v]
    for d in range(5):
        for s, step in enumerate((-1, 1)):
            e = np.zeros(6, np.int64)
            e[col[d]] = step
            hit = np.all(diff == e, axis=2)
            expect = np.where(hit.any(1), hit.argmax(1), -1)
            assert np.array_equal(g.nbr[:, 2 * d + s], expect)
    # symmetry
    for v, j in zip(*np.nonzero(g.nbr >= 0)):
        assert g.nbr[g.nbr[v, j], j ^ 1] == v


def test_frame_start():
    w = make("c1")
    rgb = np.concatenate([w.rgb, w.rgb[:, ::-1]])
    g = O.build_grid(rgb, 8.0, 8.0, 8.0)
    assert g.frame_start[0] == 0 and g.frame_start[-1] == g.M
    assert np.all(g.V[g.frame_start[1]:, 0] == 1) and np.all(g.V[:g.frame_start[1], 0] == 0)


# ----------------------------------------------------------------------------- S, B̄, Alg. 1
def test_splat_slice_identities():
    rgb, t, c, *s = tiny_case()
    g = O.build_grid(rgb, *s)
    S = O.splat_matrix(g.vid, g.M)
    # dense S by loops (brute force)
    Sd = np.zeros((g.M, g.N))
    for p in range(g.N):
        Sd[g.vid[p], p] = 1
    assert np.array_equal(S.toarray(), Sd)
    assert np.array_equal(S @ np.ones(g.N), g.m)  # S1 = m
    assert np.allclose((S @ S.T).toarray(), np.diag(g.m))  # SSᵀ = Dm
    rng = np.random.default_rng(0)
    p, v = rng.normal(size=g.N), rng.normal(size=g.M)
    assert abs((S @ p) @ v - p @ (S.T @ v)) < 1e-12 * np.abs(p).sum() * np.abs(v).max()


def test_blur_examples(worked):
    g = O.build_grid(const_image([1, 2, 3], 1, 1), 1.0, 8.0, 8.0)
    assert np.array_equal(O.blur_matrix(g.nbr) @ np.array([1.0]), [10.0])
    ex = worked["two_vertex_line"]
    g2 = O.build_grid(const_image(ex["rgb"], 1, 2), 1.0, 8.0, 8.0)
    B = O.blur_matrix(g2.nbr)
    assert np.array_equal(B @ np.array([1.0, 0.0]), [10.0, 1.0])
    rgb, *_rest = tiny_case()
    g3 = O.build_grid(rgb, 4.0, 16.0, 16.0)
    B3 = O.blur_matrix(g3.nbr)
    assert (B3 - B3.T).nnz == 0
    assert np.all(B3.diagonal() == 10)


def test_bistoch_closed_forms(worked):
    ex = worked["bistoch_closed_forms"]
    g = O.build_grid(const_image([9, 9, 9], 2, 2), 2.0, 8.0, 8.0)  # 1 vertex, m = 4
    n, res = O.bistochastize(g.m, O.blur_matrix(g.nbr), 1)
    assert n[0] == pytest.approx(ex["isolated_m4_n"], rel=1e-15)
    g2 = O.build_grid(const_image([9, 9, 9], 1, 2), 1.0, 8.0, 8.0)  # x-adjacent pair, m = 1
    n2, res2 = O.bistochastize(g2.m, O.blur_matrix(g2.nbr), 20)
    assert np.allclose(n2, ex["pair_m1_n"], rtol=1e-14) and res2 < 1e-14


def test_bistoch_converges_and_what_bistochastic():
    """Ŵ rows sum to 1 ± 1e-4, symmetric, non-negative; n∘B̄n = m (north_star)."""
    w = make("c1")
    g = O.build_grid(w.rgb, 8.0, 8.0, 8.0)
    B = O.blur_matrix(g.nbr)
    n, res = O.bistochastize(g.m, B, 20)
    assert res < 1e-8
    assert np.allclose(n * (B @ n), g.m, rtol=1e-8)
    S = O.splat_matrix(g.vid, g.M)
    What = O.dense_W_hat(S, B, g.m.astype(float), n)
    assert np.allclose(What.sum(1), 1.0, atol=1e-4)
    assert np.allclose(What, What.T) and What.min() >= 0


# ----------------------------------------------------------------------------- system
def test_one_vertex_example(worked):
    ex = worked["one_vertex"]
    rgb = const_image(ex["rgb"], ex["H"], ex["W"])
    grid, sol = frame_solve(rgb, ex["t"], ex["c"], ex["sigma_xy"], ex["sigma_l"], ex["sigma_uv"], ex["lam"],
                            mode="tol", tol=1e-14, max_iters=10)
    assert np.allclose(sol.sys.A.toarray(), ex["A"], atol=1e-15)
    assert np.allclose(sol.sys.b[:, 0], ex["b"]) and np.allclose(sol.y[:, 0], ex["y"])
    assert np.allclose(sol.x[0], ex["x"])
    dt, dc, db, _ = O.solve_backward(sol, np.array([ex["g"]]), np.array([ex["t"]]), np.array(ex["c"]),
                                     O.SolveOptions(mode="tol", tol=1e-14))
    assert np.allclose(db[:, 0], ex["d_b"]) and np.allclose(dt[0], ex["dt"]) and np.allclose(dc, ex["dc"])


def test_two_vertex_example(worked):
    ex = worked["two_vertex_line"]
    rgb = const_image(ex["rgb"], ex["H"], ex["W"])
    grid, sol = frame_solve(rgb, ex["t"], ex["c"], ex["sigma_xy"], ex["sigma_l"], ex["sigma_uv"], ex["lam"],
                            mode="tol", tol=1e-14, max_iters=10)
    assert np.allclose(sol.n, ex["n"], rtol=1e-14)
    assert np.allclose(sol.sys.A.toarray(), ex["A"], atol=1e-12)
    assert np.allclose(sol.sys.b[:, 0], ex["b"])
    assert np.allclose(sol.y[:, 0], ex["y"], atol=1e-12)
    dt, dc, db, _ = O.solve_backward(sol, np.array([ex["g"]]), np.array([ex["t"]]), np.array(ex["c"]),
                                     O.SolveOptions(mode="tol", tol=1e-14))
    assert np.allclose(db[:, 0], ex["d_b"], atol=1e-12)
    assert np.allclose(dt[0], ex["dt"], atol=1e-12) and np.allclose(dc, ex["dc"], atol=1e-12)


def _tiny_system(K=1, seed=7, **kw):
    rgb, t, c, sxy, sl, suv = tiny_case(seed=seed, K=K, **kw)
    grid, sol = frame_solve(rgb, t, c, sxy, sl, suv, 5.0, mode="tol", tol=1e-13, max_iters=5000)
    return rgb, t, c, grid, sol


def test_galerkin_and_objective_identity():
    """S(λ(I−Ŵ)+C)Sᵀ = A (derived from PAPER.md:681-704) and Eq.1(Sᵀy) = yᵀAy − 2bᵀy + (c∘t)ᵀt."""
    rgb, t, c, grid, sol = _tiny_system()
    lam = 5.0
    S = sol.S
    B = O.blur_matrix(sol.nbr)
    What = O.dense_W_hat(S, B, sol.m.astype(float), sol.n)
    N = S.shape[1]
    G = S.toarray() @ (lam * (np.eye(N) - What) + np.diag(c)) @ S.toarray().T
    assert np.allclose(G, sol.sys.A.toarray(), atol=1e-9 * lam)
    rng = np.random.default_rng(1)
    y = rng.normal(size=S.shape[0])
    x = S.T @ y
    lhs = O.pixel_loss(x, What, c, t[0], lam)
    A = sol.sys.A
    rhs = y @ (A @ y) - 2 * sol.sys.b[:, 0] @ y + (c * t[0]) @ t[0]
    assert lhs == pytest.approx(rhs, rel=1e-7)


def test_A_spd_and_dense_solve():
    rgb, t, c, grid, sol = _tiny_system()
    A = sol.sys.A.toarray()
    assert np.allclose(A, A.T)
    assert np.linalg.eigvalsh(A).min() > 0
    y_chol = sla.cho_solve(sla.cho_factor(A), sol.sys.b[:, 0])
    assert np.allclose(sol.y[:, 0], y_chol, rtol=1e-9, atol=1e-9 * np.abs(y_chol).max())


def test_c1_pcg_matches_cholesky():
    """Oracle PCG to tol 1e-12 equals the dense Cholesky solution on config 1."""
    w = make("c1")
    grid, sol = frame_solve(w.rgb, w.t[0], w.c[0], 8.0, 8.0, 8.0, 128.0, mode="tol", tol=1e-12, max_iters=5000)
    A = sol.sys.A.toarray()
    y = sla.cho_solve(sla.cho_factor(A), sol.sys.b[:, 0])
    assert np.abs(sol.y[:, 0] - y).max() <= 1e-9 * np.abs(y).max()
    # PSD/PD identity: yᵀ(Dm − DnB̄Dn)y = Σ_edges n_u n_v (y_u − y_v)² + Σ res_v y_v²
    rng = np.random.default_rng(2)
    v = rng.normal(size=A.shape[0])
    B = O.blur_matrix(sol.nbr)
    n, m = sol.n, sol.m.astype(float)
    res = m - n * (B @ n)
    quad = v @ ((np.diag(m) - np.diag(n) @ B.toarray() @ np.diag(n)) @ v)
    e = sum(n[a] * n[b] * (v[a] - v[b]) ** 2 for a, j in zip(*np.nonzero(sol.nbr >= 0)) for b in [sol.nbr[a, j]]) / 2
    assert quad == pytest.approx(e + np.sum(res * v * v), rel=1e-9)


def test_pcg_2x2(worked):
    ex = worked["pcg_2x2"]
    A = np.array(ex["A"])
    r = O.pcg(lambda v: A @ v, np.array(ex["b"]), np.zeros(2), lambda v: v, 2)
    assert np.allclose(r.x, ex["y"], atol=1e-14) and r.iterations == 2
    r2 = O.pcg(lambda v: A @ v, np.array(ex["b"]), np.zeros(2), lambda v: v / np.diag(A), 2)
    assert np.allclose(r2.x, ex["y"], atol=1e-14)
    r3 = O.pcg(lambda v: v, np.array(ex["b"]), np.zeros(2), lambda v: v, 5, tol=1e-12)
    assert r3.iterations == 1 and np.allclose(r3.x, ex["b"])  # identity → 1 iteration


def test_pcg_random_spd_and_monotone_loss():
    rng = np.random.default_rng(11)
    for n in (5, 40, 120):
        Q = rng.normal(size=(n, n))
        A = Q @ Q.T + n * np.eye(n)
        b = rng.normal(size=n)
        r = O.pcg(lambda v: A @ v, b, np.zeros(n), lambda v: v / np.diag(A), n + 20, tol=1e-12, track_loss=True)
        assert np.allclose(r.x, np.linalg.solve(A, b), rtol=1e-8, atol=1e-10)
        L = np.array(r.losses)
        assert np.all(np.diff(L) <= 1e-9 * np.abs(L).max())


def test_pcg_tol_stop_rule_and_fixed_count():
    A = np.diag([1.0, 10.0, 100.0])
    b = np.ones(3)
    r = O.pcg(lambda v: A @ v, b, np.linalg.solve(A, b), lambda v: v, 50, tol=1e-6)
    assert r.iterations == 0  # tested before iteration 0 (reading #11)
    r = O.pcg(lambda v: A @ v, np.zeros(3), np.zeros(3), lambda v: v, 50, tol=1e-6)
    assert r.iterations == 0  # ‖b‖ = 0 → converged at i = 0
    r = O.pcg(lambda v: A @ v, b, np.zeros(3), lambda v: v, 2)
    assert r.iterations == 2


def test_solver_invariants():
    rgb, t, c, sxy, sl, suv = tiny_case(K=1)
    HW = t.shape[1]
    # constant target → constant output (north_star invariant)
    _, s = frame_solve(rgb, np.full((1, HW), 3.25), c, sxy, sl, suv, 50.0, mode="tol", tol=1e-13, max_iters=5000)
    assert np.allclose(s.x, 3.25, atol=1e-8)
    # (c, λ) → (κc, κλ) leaves y unchanged
    _, s1 = frame_solve(rgb, t, c, sxy, sl, suv, 7.0, mode="tol", tol=1e-13, max_iters=5000)
    _, s2 = frame_solve(rgb, t, 3.0 * c, sxy, sl, suv, 21.0, mode="tol", tol=1e-13, max_iters=5000)
    assert np.allclose(s1.y, s2.y, atol=1e-9)
    # linear in t (fixed c)
    t2 = np.random.default_rng(5).normal(size=t.shape)
    _, sa = frame_solve(rgb, t2, c, sxy, sl, suv, 7.0, mode="tol", tol=1e-13, max_iters=5000)
    _, sb = frame_solve(rgb, 2 * t - 3 * t2, c, sxy, sl, suv, 7.0, mode="tol", tol=1e-13, max_iters=5000)
    assert np.allclose(sb.y, 2 * s1.y - 3 * sa.y, atol=1e-8)


def test_lambda_to_zero_limit():
    """Reading #16: λ→0 gives y = b/Sc (flat init); with t = f(vid), x → t where c > 0."""
    rgb, t, c, sxy, sl, suv = tiny_case(K=1)
    grid, s = frame_solve(rgb, t, c, sxy, sl, suv, 1e-9, mode="tol", tol=1e-14, max_iters=5000)
    assert np.allclose(s.y, O.flat_init(s.sys), atol=1e-7)
    tv = np.random.default_rng(4).uniform(size=grid.M)[grid.vid][None]
    _, s2 = frame_solve(rgb, tv, c, sxy, sl, suv, 1e-9, mode="tol", tol=1e-14, max_iters=5000)
    assert np.allclose(s2.x, tv, atol=1e-7)


def test_flat_init_and_dead_vertex():
    """Eq. flat_init with the Sc = 0 → 0 rule (reading #9) and the dead-vertex rule (reading #6)."""
    rgb = const_image([10, 10, 10], 1, 3)
    rgb[0, 0, 2] = [250, 250, 250]  # isolated vertex (different luma, not adjacent in l)
    t = np.array([[1.0, 2.0, 5.0]])
    c = np.array([1.0, 3.0, 0.0])
    grid, s = frame_solve(rgb, t, c, 2.0, 8.0, 8.0, 4.0, mode="tol", tol=1e-12, max_iters=100)
    assert grid.M == 2 and np.all(grid.nbr < 0)
    assert np.allclose(O.flat_init(s.sys)[:, 0], [(1 * 1 + 3 * 2) / 4.0, 0.0])
    assert list(s.sys.live) == [True, False]
    assert np.all(np.isfinite(s.y)) and s.y[1, 0] == 0.0


# ----------------------------------------------------------------------------- pyramid / hierarchical
def test_z_weight(paper_params):
    for case in paper_params["z_weight"]["cases"]:
        assert O.z_weight(case["k"], case["alpha"], case["beta"]) == case["value"]


def test_pyramid_bruteforce():
    """Level k = unique(⌊V/2^k⌋) (independent: one floor-division by 2^k), parents consistent,
    P(1) = subtree counts, top level a single vertex."""
    w = make("c1")
    g = O.build_grid(w.rgb, 8.0, 8.0, 8.0)
    pyr = O.build_pyramid(g.V)
    assert pyr.levels[-1].shape[0] == 1
    assert all(pyr.levels[k + 1].shape[0] < pyr.levels[k].shape[0] for k in range(pyr.K - 1))
    for k in range(pyr.K):
        Vk = g.V.copy()
        Vk[:, 1:] //= 2 ** k
        assert np.array_equal(np.unique(Vk, axis=0), pyr.levels[k])
    P1 = O.P_lift(pyr, np.ones(g.M))
    for k in range(1, pyr.K):
        Vk = g.V.copy()
        Vk[:, 1:] //= 2 ** k
        cnt = [np.sum(np.all(Vk == row, axis=1)) for row in pyr.levels[k]]
        assert np.array_equal(P1[k], cnt)
        # parents map children onto the halved tuple
        H = pyr.levels[k - 1].copy()
        H[:, 1:] //= 2
        assert np.array_equal(pyr.levels[k][pyr.parents[k - 1]], H)


def test_P_adjoint():
    w = make("c1")
    g = O.build_grid(w.rgb, 8.0, 8.0, 8.0)
    pyr = O.build_pyramid(g.V)
    rng = np.random.default_rng(8)
    y = rng.normal(size=g.M)
    z = [rng.normal(size=L.shape[0]) for L in pyr.levels]
    lhs = sum(a @ b for a, b in zip(O.P_lift(pyr, y), z))
    assert lhs == pytest.approx(y @ O.P_project(pyr, z), rel=1e-12)


def test_hier_4x1_closed_form(worked):
    ex = worked["hier_4x1_line"]
    rgb = const_image(ex["rgb"], ex["H"], ex["W"])
    rng = np.random.default_rng(2)
    c = rng.uniform(0.5, 1.5, 4)
    grid, s = frame_solve(rgb, np.zeros((1, 4)), c, ex["sigma_xy"], ex["sigma_l"], ex["sigma_uv"], 3.0,
                          precond="hier", init="hier", mode="fixed", iters=1)
    assert [L.shape[0] for L in s.pyr.levels] == ex["level_sizes"]
    dA = s.sys.diagA
    e0 = np.array([1.0, 0, 0, 0])
    expect = e0 / dA[0] + ex["w1"] * 2 / (dA[0] + dA[1]) * np.array([1, 1, 0, 0]) \
        + ex["w2"] * 4 / dA.sum() * np.ones(4)
    assert np.allclose(s.Minv(e0), expect, rtol=1e-14)


def test_hier_init_4x1_closed_form(worked):
    """y_hier at the paper's α = 4, β = 0 on the 4×1 line, against the closed
    form derived by hand in tests/golden (each vertex one pixel: b = c∘t, Sc = c).  Every coarse
    term is live here, so P(1) multiplied instead of divided, a shifted level index in z_w, a
    dropped level or swapped numerator/denominator all fail."""
    ex = worked["hier_init_4x1_line"]
    rgb = const_image(ex["rgb"], ex["H"], ex["W"])
    rng = np.random.default_rng(21)
    c = rng.uniform(0.2, 1.5, 4)
    t = rng.uniform(-3.0, 5.0, (1, 4))
    _, s = frame_solve(rgb, t, c, ex["sigma_xy"], ex["sigma_l"], ex["sigma_uv"], 3.0,
                       precond="jacobi", init="hier", mode="fixed", iters=0)
    b, Sc = c * t[0], c
    w1, w2 = ex["w1"], ex["w2"]
    expect = np.empty(4)
    for v, (p0, p1) in enumerate(ex["pairs"]):
        num = b[v] + w1 * (b[p0] + b[p1]) / 2 + w2 * b.sum() / 4
        den = Sc[v] + w1 * (Sc[p0] + Sc[p1]) / 2 + w2 * Sc.sum() / 4
        expect[v] = num / den
    assert np.allclose(s.y0[:, 0], expect, rtol=1e-14, atol=0)
    assert np.allclose(s.y[:, 0], expect, rtol=1e-14, atol=0)  # 0 PCG iterations


def test_diagA_closed_forms(worked):
    """diag(A): (a) the 2-vertex worked example's diagonal [2, 2]; (b) it equals
    the diagonal of the explicitly assembled sparse A; (c) at Alg. 1's fixed point n∘B̄n = m it
    equals λ n_v Σ_{u∈N(v)} n_u + Sc_v (the edge-weight form — an independent route through the
    neighbour lists), up to λ × the bistochastization residual."""
    ex = worked["two_vertex_line"]
    rgb = const_image(ex["rgb"], ex["H"], ex["W"])
    _, s = frame_solve(rgb, [ex["t"]], ex["c"], ex["sigma_xy"], ex["sigma_l"], ex["sigma_uv"], ex["lam"])
    assert np.allclose(s.sys.diagA, np.diag(ex["A"]), rtol=1e-12)
    rgb, t, c, sxy, sl, suv = tiny_case(seed=5)
    lam = 7.0
    grid = O.build_grid(rgb, sxy, sl, suv)
    s = O.solve_frame(grid, 0, t, c, lam, O.SolveOptions(mode="fixed", iters=0, n_bistoch=80))
    assert np.allclose(s.sys.diagA, s.sys.A.diagonal(), rtol=1e-13, atol=1e-13)
    nsum = np.array([sum(s.n[u] for u in row if u >= 0) for row in s.nbr])
    Sc_direct = np.bincount(s.vid, weights=c, minlength=grid.M)
    closed = lam * s.n * nsum + Sc_direct
    assert s.bistoch_residual < 1e-12
    assert np.abs(s.sys.diagA - closed).max() <= 1e-9 * lam * s.m.max()
    assert np.sum(nsum > 0) > 0.5 * grid.M  # most vertices have neighbours: the test has teeth


def test_hier_degenerations():
    """α → ∞: hier precond → Jacobi, hier init → flat; M = 1 → Jacobi."""
    rgb, t, c, sxy, sl, suv = tiny_case(K=2)
    grid = O.build_grid(rgb, sxy, sl, suv)
    s = O.solve_frame(grid, 0, t, c, 5.0, O.SolveOptions(precond="hier", init="hier", mode="fixed", iters=0))
    pyr, sysm = s.pyr, s.sys
    Mh = O.hier_minv(pyr, sysm, 1e6, 5.0)
    Mj = O.jacobi_minv(sysm)
    r = np.random.default_rng(0).normal(size=grid.M)
    assert np.allclose(Mh(r), Mj(r), rtol=1e-4, atol=1e-4 * np.abs(Mj(r)).max())
    yi = O.hier_init(pyr, sysm, 1e8, 0.0)  # error O(1/α)
    assert np.allclose(yi, O.flat_init(sysm), atol=1e-6)
    # symmetric and PD probes
    M2 = O.hier_minv(pyr, sysm, 2.0, 5.0)
    u, v = np.random.default_rng(1).normal(size=(2, grid.M))
    assert M2(u) @ v == pytest.approx(u @ M2(v), rel=1e-10)
    assert M2(u) @ u > 0
    # M = 1
    g1 = O.build_grid(const_image([5, 5, 5], 2, 2), 2.0, 8.0, 8.0)
    s1 = O.solve_frame(g1, 0, np.ones((1, 4)), np.ones(4), 1.0, O.SolveOptions(precond="hier", init="hier"))
    assert s1.pyr.K == 1
    assert np.allclose(s1.Minv(np.array([2.0])), O.jacobi_minv(s1.sys)(np.array([2.0])))


def test_hier_solution_equals_jacobi_solution():
    """Preconditioner / init change the path, not the minimiser."""
    rgb, t, c, sxy, sl, suv = tiny_case(K=1)
    _, a = frame_solve(rgb, t, c, sxy, sl, suv, 9.0, precond="hier", init="hier", mode="tol", tol=1e-13,
                       max_iters=5000)
    _, b = frame_solve(rgb, t, c, sxy, sl, suv, 9.0, precond="jacobi", init="flat", mode="tol", tol=1e-13,
                       max_iters=5000)
    assert np.allclose(a.x, b.x, atol=1e-8)


# ----------------------------------------------------------------------------- backward
def test_backward_linearity_identity():
    """x is linear in t, so ⟨∂t, δ⟩ = ⟨g, x(t+δ) − x(t)⟩ exactly."""
    rgb, t, c, sxy, sl, suv = tiny_case(K=2)
    opts = dict(mode="tol", tol=1e-14, max_iters=5000)
    grid, s = frame_solve(rgb, t, c, sxy, sl, suv, 6.0, **opts)
    rng = np.random.default_rng(9)
    g = rng.normal(size=t.shape)
    delta = rng.normal(size=t.shape)
    dt, dc, db, _ = O.solve_backward(s, g, t, c, O.SolveOptions(**opts))
    _, s2 = frame_solve(rgb, t + delta, c, sxy, sl, suv, 6.0, **opts)
    assert np.sum(dt * delta) == pytest.approx(np.sum(g * (s2.x - s.x)), rel=1e-8)


def test_backward_dc_finite_difference():
    """∂f/∂c by central differences (h = 1e-4, fp64), f(x̂) = ⟨g, x̂⟩."""
    rgb, t, c, sxy, sl, suv = tiny_case(K=2, W=12, H=10, sxy=3.0)
    opts = dict(mode="tol", tol=1e-14, max_iters=5000)
    grid, s = frame_solve(rgb, t, c, sxy, sl, suv, 6.0, **opts)
    g = np.random.default_rng(10).normal(size=t.shape)
    dt, dc, db, _ = O.solve_backward(s, g, t, c, O.SolveOptions(**opts))
    h = 1e-4
    for p in np.random.default_rng(12).choice(c.size, 32, replace=False):
        cp, cm = c.copy(), c.copy()
        cp[p] += h
        cm[p] -= h
        _, sp_ = frame_solve(rgb, t, cp, sxy, sl, suv, 6.0, **opts)
        _, sm_ = frame_solve(rgb, t, cm, sxy, sl, suv, 6.0, **opts)
        fd = (np.sum(g * sp_.x) - np.sum(g * sm_.x)) / (2 * h)
        assert abs(fd - dc[p]) <= 1e-4 * (abs(dc[p]) + 1e-6) + 1e-8
    for p in np.random.default_rng(13).choice(c.size, 8, replace=False):
        for k in range(2):
            tp, tm = t.copy(), t.copy()
            tp[k, p] += h
            tm[k, p] -= h
            _, sp_ = frame_solve(rgb, tp, c, sxy, sl, suv, 6.0, **opts)
            _, sm_ = frame_solve(rgb, tm, c, sxy, sl, suv, 6.0, **opts)
            fd = (np.sum(g * sp_.x) - np.sum(g * sm_.x)) / (2 * h)
            assert abs(fd - dt[k, p]) <= 1e-4 * (abs(dt[k, p]) + 1e-6) + 1e-8


def test_zero_confidence_components():
    rgb = const_image([10, 10, 10], 1, 4)
    rgb[0, 0, 2:] = [250, 250, 250]  # second component (x = 2, 3), σxy = 1
    grid, s = frame_solve(rgb, np.ones((1, 4)), np.array([1.0, 1.0, 0.0, 0.0]), 1.0, 8.0, 8.0, 1.0,
                          mode="fixed", iters=3)
    zc = O.zero_confidence_components(s.nbr, s.sys.Sc)
    assert list(zc) == [False, False, True, True]


def test_multichannel_equals_separate_solves():
    rgb, t, c, sxy, sl, suv = tiny_case(K=3)
    opts = dict(mode="fixed", iters=7, precond="hier", init="hier")
    _, s = frame_solve(rgb, t, c, sxy, sl, suv, 4.0, **opts)
    for k in range(3):
        _, sk = frame_solve(rgb, t[k:k + 1], c, sxy, sl, suv, 4.0, **opts)
        assert np.allclose(sk.x[0], s.x[k], atol=1e-12)
