"""Reading #29's premise, pinned on the CPU (no GPU involved): at a fixed count of 25 PCG
iterations on the bench workload (configs[4], frame 0, full 1920×1080 size), the fp64 oracle's
own iterate is unstable at a handful of pixels (single-pixel vertices with ≤ 1 neighbour) — perturbing the PCG vectors by a relative 1e-8
moves those pixels by more than half the north_star bound, and nowhere else does the iterate move
by more than a small fraction of it.  The GPU parity test exempts exactly the pixels where fp32
vector storage moves the oracle's iterate (tests/parity_util.fixed_count_unstable) and bounds
their count by 1e-5 of the pixels; this test shows that set is the oracle's own instability, not
an implementation error, and keeps its size pinned."""
import numpy as np
import pytest

import oracle as O
from parity_util import MAX_TOL, fixed_count_unstable, oracle_opts, target_range
from workloads import make


def pcg_perturbed(sol, iters, rel, seed, k=0):
    """Alg. 2 with the oracle's operators, every vector multiplied by
    (1 + rel·ξ), ξ ~ N(0, 1), right after it is formed.  Returns the sliced result of channel k."""
    rng = np.random.default_rng(seed)
    pert = lambda v: v * (1.0 + rel * rng.standard_normal(v.shape))  # noqa: E731
    A, Minv = sol.sys.A, sol.Minv
    b = sol.sys.b[:, k]
    x = pert(sol.y0[:, k].astype(np.float64))
    r = pert(b - A @ x)
    d = pert(Minv(r))
    rho = float(r @ d)
    for _ in range(iters):
        q = pert(A @ d)
        alpha = rho / float(d @ q)
        x = pert(x + alpha * d)
        r = pert(r - alpha * q)
        s = pert(Minv(r))
        rho_old, rho = rho, float(r @ s)
        d = pert(s + (rho / rho_old) * d)
    return x[sol.vid]


@pytest.fixture(scope="module")
def frame0():
    w = make("c5", frames=1)
    _, sols = O.solve(w.rgb, w.t, w.c, w.sigma_xy, w.sigma_l, w.sigma_uv, w.lam, oracle_opts(w))
    HW = w.H * w.W
    return w, sols[0], w.t[0].reshape(1, HW).astype(np.float64), w.c[0].reshape(HW).astype(np.float64)


def test_fixed_count_iterate_is_unstable_at_few_pixels(frame0):
    w, sol, t, c = frame0
    rng_t = target_range(t, c)[0]
    HW = t.shape[1]
    half = 0.5 * MAX_TOL * rng_t
    moved_sets = []
    for seed in (1, 2, 3):
        xp = pcg_perturbed(sol, w.iters, 1e-8, seed)
        dev = np.abs(xp - sol.x[0])
        moved = dev > half
        moved_sets.append(moved)
        # the instability exists (the premise) and is confined to a handful of pixels
        assert 1 <= moved.sum() <= 1e-5 * HW, moved.sum()
        # everywhere else the perturbed iterate stays far inside the bound
        assert dev[~moved].max() <= half
        assert np.sqrt(np.mean(dev ** 2)) <= 1e-4 * rng_t  # RMS over all pixels within the bound
    # the set does not depend on the perturbation: the same pixels move under every draw
    assert np.array_equal(moved_sets[0], moved_sets[1]) and np.array_equal(moved_sets[0], moved_sets[2])
    # and it is the set the GPU test exempts (fp32 storage is a perturbation of the same kind)
    unstable, _ = fixed_count_unstable(sol, w.iters, t, c)
    assert unstable.sum() <= 1e-5 * HW
    assert (unstable & moved_sets[0]).sum() >= 1
    # the unstable pixels are single-pixel vertices with at most one neighbour (tiny, weakly
    # coupled components whose Krylov components converge last)
    v = sol.vid[moved_sets[0] | unstable]
    assert np.all(sol.m[v] == 1) and np.all((sol.nbr[v] >= 0).sum(axis=1) <= 1)
    # the amplification is a property of the iterate: a 1e-12 perturbation moves nothing visibly
    xp = pcg_perturbed(sol, w.iters, 1e-12, 4)
    assert np.abs(xp - sol.x[0]).max() <= 1e-5 * rng_t
