"""Seeded synthetic inputs standing in for the paper's (unavailable) datasets.

The paper measures on Barron 2015A's 4-MP profiling images,
Middlebury / Ferstl depth super-resolution and Pascal
VOC segmentation maps; none is in the container.  The
generators below reproduce the *structure* of those workloads as BASELINE.json
``configs`` describe them: piecewise-smooth Voronoi reference images with
gradients and Gaussian noise, planar depth targets with outliers, sparse
super-resolution samples and 21-channel class probabilities.

Draw order (numpy ``default_rng(seed)``, PCG64), per reference image:
  1. seeds          n_cells x 2   uniform [0, W) x [0, H)
  2. base colours   n_cells x 3   U(0, 255)
  3. slopes         n_cells x 3 x 2  U(-0.5, 0.5) per px   (mode == "gradient")
  4. noise          H x W x 3     N(0, sigma_noise^2)
then target/confidence draws continue from the same generator.
Pixel centre (x + 1/2, y + 1/2) takes the label of its nearest seed.
Colours are rounded half-to-even, clipped to [0, 255] and stored as uint8.

Nothing here implements the bilateral solver; see oracle/ and the CUDA path.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np
from scipy.spatial import cKDTree


@dataclass
class Workload:
    """One solve: F frames of (reference, target, confidence) + solver settings.

    Layouts (the C-ABI's, include/fbs.h):
      rgb : uint8   [F][H][W][3]  interleaved RGB
      t   : float32 [F][K][H][W]  planar targets
      c   : float32 [F][H][W]     confidence >= 0
      g   : float32 [F][K][H][W]  upstream gradient dL/dx (backward configs)
    """

    name: str
    rgb: np.ndarray
    t: np.ndarray
    c: np.ndarray
    sigma_xy: float
    sigma_l: float
    sigma_uv: float
    lam: float
    precond: str = "jacobi"  # "jacobi" | "hier"
    init: str = "flat"  # "flat" | "hier"
    mode: str = "tol"  # "tol" | "fixed"
    iters: int = 25
    tol: float = 1e-6
    max_iters: int = 2000
    n_bistoch: int = 20
    g: Optional[np.ndarray] = None
    labels: Optional[np.ndarray] = field(default=None, repr=False)
    truth: Optional[np.ndarray] = field(default=None, repr=False)  # clean target (robust configs)
    sigma_gm: float = 0.0  # robust configs: Geman–McClure scale
    n_irls: int = 0  # robust configs: IRLS iterations

    @property
    def frames(self) -> int:
        return self.rgb.shape[0]

    @property
    def H(self) -> int:
        return self.rgb.shape[1]

    @property
    def W(self) -> int:
        return self.rgb.shape[2]

    @property
    def K(self) -> int:
        return self.t.shape[1]

    @property
    def pixels(self) -> int:
        return self.frames * self.H * self.W


def _labels(seeds: np.ndarray, W: int, H: int) -> np.ndarray:
    """Nearest-seed label of every pixel centre, int32 [H][W]."""
    ys, xs = np.mgrid[0:H, 0:W]
    centres = np.stack([xs.ravel() + 0.5, ys.ravel() + 0.5], axis=1)
    _, lab = cKDTree(seeds).query(centres, k=1)
    return lab.reshape(H, W).astype(np.int32)


def voronoi_reference(rng, W, H, n_cells, mode, sigma_noise):
    """Piecewise (constant | linear-gradient) Voronoi RGB image + labels + seeds."""
    seeds = np.stack([rng.uniform(0, W, n_cells), rng.uniform(0, H, n_cells)], axis=1)
    base = rng.uniform(0, 255, (n_cells, 3))
    slopes = rng.uniform(-0.5, 0.5, (n_cells, 3, 2)) if mode == "gradient" else None
    noise = rng.normal(0.0, sigma_noise, (H, W, 3))
    lab = _labels(seeds, W, H)
    img = base[lab].copy()
    if slopes is not None:
        ys, xs = np.mgrid[0:H, 0:W]
        dx = xs + 0.5 - seeds[lab, 0]
        dy = ys + 0.5 - seeds[lab, 1]
        img += slopes[lab, :, 0] * dx[..., None] + slopes[lab, :, 1] * dy[..., None]
    img += noise
    rgb = np.clip(np.rint(img), 0, 255).astype(np.uint8)
    return rgb, lab, seeds


def planar_depth(rng, lab, seeds):
    """Per-region random plane in [0, 255]: d0 ~ U(0,255) at the seed, slopes U(-0.1, 0.1)."""
    n = seeds.shape[0]
    H, W = lab.shape
    d0 = rng.uniform(0, 255, n)
    s = rng.uniform(-0.1, 0.1, (n, 2))
    ys, xs = np.mgrid[0:H, 0:W]
    d = d0[lab] + s[lab, 0] * (xs + 0.5 - seeds[lab, 0]) + s[lab, 1] * (ys + 0.5 - seeds[lab, 1])
    return np.clip(d, 0, 255)


def _depth_with_outliers(rng, lab, seeds, frac):
    d = planar_depth(rng, lab, seeds)
    H, W = lab.shape
    out = rng.uniform(0, 1, (H, W)) < frac
    d = np.where(out, rng.uniform(0, 255, (H, W)), d)
    c = np.where(out, rng.uniform(0, 0.2, (H, W)), rng.uniform(0.6, 1.0, (H, W)))
    return d, c


# --------------------------------------------------------------------------- configs


def c1_tiny(W=64, H=48, seed=1001):
    """BASELINE.json configs[0]: 64x48, 12 constant Voronoi cells + N(0,4^2)."""
    rng = np.random.default_rng(seed)
    rgb, lab, seeds = voronoi_reference(rng, W, H, 12, "constant", 4.0)
    val = rng.uniform(0, 1, 12)
    t = val[lab] + rng.normal(0, 0.05, (H, W))
    c = rng.uniform(0.1, 1.0, (H, W))
    return Workload("c1_tiny", rgb[None], t[None, None].astype(np.float32), c[None].astype(np.float32),
                    8.0, 8.0, 8.0, 128.0, precond="jacobi", init="flat", mode="tol", tol=1e-6,
                    labels=lab[None])


def c2_depth_refine(W=1390, H=1110, seed=1002, n_cells=200):
    """configs[1]: depth refinement, 10% outliers, hier precond + init."""
    rng = np.random.default_rng(seed)
    rgb, lab, seeds = voronoi_reference(rng, W, H, n_cells, "gradient", 3.0)
    d, c = _depth_with_outliers(rng, lab, seeds, 0.10)
    return Workload("c2_depth_refine", rgb[None], d[None, None].astype(np.float32),
                    c[None].astype(np.float32), 8.0, 4.0, 3.0, 128.0,
                    precond="hier", init="hier", mode="tol", tol=1e-6, labels=lab[None])


def c3_depth_sr(H=1088, W=1376, seed=1003, n_cells=200, stride=16):
    """configs[2]: depth super-resolution, target known on every 16th px (c=1), else t=c=0.

    Shape reading: numpy (H, W) = (1088, 1376)."""
    rng = np.random.default_rng(seed)
    rgb, lab, seeds = voronoi_reference(rng, W, H, n_cells, "gradient", 3.0)
    d = planar_depth(rng, lab, seeds)
    known = np.zeros((H, W), bool)
    known[::stride, ::stride] = True
    t = np.where(known, d, 0.0)
    c = known.astype(np.float64)
    return Workload("c3_depth_sr", rgb[None], t[None, None].astype(np.float32), c[None].astype(np.float32),
                    8.0, 4.0, 4.0, 256.0, precond="hier", init="hier", mode="fixed", iters=25,
                    tol=1e-6, labels=lab[None])


def c4_multichannel(W=500, H=375, seed=1004, n_cells=60, K=21, grad_seed=1104):
    """configs[3]: 21-channel class probabilities solved jointly, then backward on g ~ N(0,1)."""
    rng = np.random.default_rng(seed)
    rgb, lab, seeds = voronoi_reference(rng, W, H, n_cells, "gradient", 3.0)
    probs = rng.dirichlet(0.3 * np.ones(K), n_cells)  # [cells][K]
    t = probs[lab] + rng.normal(0, 0.02, (H, W, K))
    t = np.clip(t, 0, None)
    s = t.sum(axis=2, keepdims=True)
    t = np.where(s > 0, t / np.where(s > 0, s, 1), 1.0 / K)
    c = rng.uniform(0.3, 1.0, (H, W))
    g = np.random.default_rng(grad_seed).normal(0, 1, (K, H, W))
    return Workload("c4_multichannel", rgb[None], np.ascontiguousarray(t.transpose(2, 0, 1))[None].astype(np.float32),
                    c[None].astype(np.float32), 8.0, 4.0, 4.0, 64.0, precond="jacobi", init="flat",
                    mode="tol", tol=1e-6, g=g[None].astype(np.float32), labels=lab[None])


def c5_batch(frames=8, W=1920, H=1080, first_frame=0, n_cells=300):
    """configs[4]: independent 1920x1080 frames (seed 5000+f), 5% outliers, hier, fixed 25."""
    rgbs, ts, cs, labs = [], [], [], []
    for f in range(first_frame, first_frame + frames):
        rng = np.random.default_rng(5000 + f)
        rgb, lab, seeds = voronoi_reference(rng, W, H, n_cells, "gradient", 3.0)
        d, c = _depth_with_outliers(rng, lab, seeds, 0.05)
        rgbs.append(rgb)
        ts.append(d[None].astype(np.float32))
        cs.append(c.astype(np.float32))
        labs.append(lab)
    return Workload("c5_batch", np.stack(rgbs), np.stack(ts), np.stack(cs), 8.0, 4.0, 3.0, 128.0,
                    precond="hier", init="hier", mode="fixed", iters=25, tol=1e-6,
                    labels=np.stack(labs))


def rbs_depth(W=640, H=480, seed=1006, n_cells=120, frac=0.10, frames=1, n_irls=8):
    """Robust bilateral solver workload (Supp. §3): piecewise-planar depth
    with a fraction of uniform outliers that the confidence does NOT flag (c_init = 1), so the
    IRLS weights must find them; `truth` is the clean depth.  Stand-in for the Middlebury stereo
    post-processing experiment, whose MC-CNN depth maps are not available."""
    rgbs, ts, cs, tr = [], [], [], []
    for f in range(frames):
        rng = np.random.default_rng(seed + 100 * f)
        rgb, lab, seeds = voronoi_reference(rng, W, H, n_cells, "gradient", 3.0)
        d = planar_depth(rng, lab, seeds)
        out = rng.uniform(0, 1, (H, W)) < frac
        t = np.where(out, rng.uniform(0, 255, (H, W)), d)
        rgbs.append(rgb)
        ts.append(t[None].astype(np.float32))
        cs.append(np.ones((H, W), np.float32))
        tr.append(d.astype(np.float32))
    return Workload("rbs_depth", np.stack(rgbs), np.stack(ts), np.stack(cs), 8.0, 4.0, 3.0, 128.0,
                    precond="hier", init="hier", mode="fixed", iters=25, tol=1e-6,
                    truth=np.stack(tr), sigma_gm=10.0, n_irls=n_irls)


CONFIGS = {
    "c1": c1_tiny,
    "c2": c2_depth_refine,
    "c3": c3_depth_sr,
    "c4": c4_multichannel,
    "c5": c5_batch,
    "rbs": rbs_depth,
}


def make(name: str, **kw) -> Workload:
    """Build a named config; keyword overrides shrink it (W, H, frames, ...) for fast tests."""
    return CONFIGS[name](**kw)
