"""Thin ctypes binding of include/fbs.h — argument marshalling only.

Every step of the bilateral-space solve runs in libfbs.so's sm_100a kernels; this module
checks tensor dtypes/devices/layouts, passes raw device pointers and the current CUDA
stream, and turns FBS_E* codes into exceptions.  There is no CPU fallback: if the
library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# FBS_LIB: an alternative in-tree build of the same library (same-box A/B measurements)
LIB_PATH = os.environ.get("FBS_LIB") or os.path.join(_HERE, "libfbs.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing — build it with `python paper_1511_03296_b200/build.py` "
                      "(the product path has no CPU fallback)")
_lib = C.CDLL(LIB_PATH)

FBS_OK, FBS_EINVAL, FBS_ENOMEM, FBS_ECUDA, FBS_ELIMIT, FBS_ESTATE = range(6)
FBS_ST_BREAKDOWN, FBS_ST_NOTCONVERGED, FBS_ST_NEG_CONF, FBS_ST_NONFINITE = 1, 2, 4, 8
PRECOND = {"jacobi": 0, "hier": 1}
INIT = {"flat": 0, "hier": 1, "zero": 2}
MODE = {"fixed": 0, "tol": 1}


class GridOpts(C.Structure):
    _fields_ = [("n_bistoch", C.c_int), ("build_pyramid", C.c_int), ("dims", C.c_int)]


class SolveOpts(C.Structure):
    _fields_ = [("precond", C.c_int), ("init", C.c_int), ("mode", C.c_int), ("iters", C.c_int),
                ("tol", C.c_double), ("max_iters", C.c_int), ("precond_alpha", C.c_double),
                ("precond_beta", C.c_double), ("init_alpha", C.c_double), ("init_beta", C.c_double),
                ("lowrank_eps", C.c_double)]


_ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
_FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)


class Allocator(C.Structure):
    _fields_ = [("alloc", _ALLOC_FN), ("free", _FREE_FN), ("ctx", C.c_void_p)]


_vp, _i, _d, _i64 = C.c_void_p, C.c_int, C.c_double, C.c_int64
_SIGS = {
    "fbs_default_grid_opts": (None, [C.POINTER(GridOpts)]),
    "fbs_default_solve_opts": (None, [C.POINTER(SolveOpts)]),
    "fbs_grid_build": (_i, [_vp, _i, _i, _i, _d, _d, _d, C.POINTER(GridOpts), _vp, C.POINTER(_vp)]),
    "fbs_grid_info": (_i, [_vp, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i), _vp, _vp, _vp]),
    "fbs_grid_export": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "fbs_pyramid_export": (_i, [_vp, _i, _vp, _vp, _vp]),
    "fbs_grid_destroy": (None, [_vp]),
    "fbs_solve": (_i, [_vp, _vp, _i, _vp, _d, C.POINTER(SolveOpts), _vp, _vp, C.POINTER(_vp), _vp]),
    "fbs_solve_robust": (_i, [_vp, _vp, _i, _vp, _d, C.POINTER(SolveOpts), _d, _i, _vp, _vp, _vp]),
    "fbs_solve_backward": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "fbs_dt_filter": (_i, [_vp, _i, _i, _i, _vp, _i, _d, _d, _i, _vp, _vp]),
    "fbs_system_stats": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "fbs_system_export": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "fbs_system_destroy": (None, [_vp]),
    "fbs_slice": (_i, [_vp, _vp, _i, _vp, _vp]),
    "fbs_splat": (_i, [_vp, _vp, _i, _vp, _vp]),
    "fbs_blur": (_i, [_vp, _vp, _vp, _vp]),
    "fbs_system_apply_A": (_i, [_vp, _vp, _vp, _vp]),
    "fbs_system_apply_precond": (_i, [_vp, _vp, _vp, _vp]),
    "fbs_last_error": (C.c_char_p, []),
    "fbs_version": (_i, []),
    "fbs_set_allocator": (_i, [C.POINTER(Allocator)]),
    "fbs_launch_count": (_i64, []),
    "fbs_profile_enable": (_i, [_i]),
    "fbs_profile_report": (_i, [C.c_char_p, C.c_size_t]),
    "fbs_profile_reset": (_i, []),
}
for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(_lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


class FbsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[fbs code {code}] {msg}")
        self.code = code


def _check(code: int):
    if code != FBS_OK:
        raise FbsError(code, _lib.fbs_last_error().decode())


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _np_ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _stream(stream) -> C.c_void_p:
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def _dev_tensor(x: torch.Tensor, dtype: torch.dtype, name: str, ndim: int) -> torch.Tensor:
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if x.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {x.dtype}")
    if x.dim() != ndim:
        raise ValueError(f"{name} must have {ndim} dims, got shape {tuple(x.shape)}")
    return x.contiguous()


def _out_tensor(out: Optional[torch.Tensor], like: torch.Tensor, name: str = "out") -> torch.Tensor:
    """A caller-supplied output buffer must be exactly what the kernels write: CUDA float32,
    contiguous, the shape of `like`, on `like`'s device (the C side cannot check any of this)."""
    if out is None:
        return torch.empty_like(like)
    if not isinstance(out, torch.Tensor) or not out.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if out.dtype != torch.float32:
        raise TypeError(f"{name} must be torch.float32, got {out.dtype}")
    if tuple(out.shape) != tuple(like.shape):
        raise ValueError(f"{name} must have shape {tuple(like.shape)}, got {tuple(out.shape)}")
    if not out.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if out.device != like.device:
        raise ValueError(f"{name} is on {out.device}, the inputs on {like.device}")
    return out


def launch_count() -> int:
    """Kernels launched by libfbs.so in this process (monotone)."""
    return int(_lib.fbs_launch_count())


def version() -> int:
    return int(_lib.fbs_version())


def profile_enable(on: bool = True):
    """Bracket every library kernel launch with CUDA events (per-kernel device timing)."""
    _lib.fbs_profile_enable(int(bool(on)))


def profile_reset():
    _check(_lib.fbs_profile_reset())


def profile_report() -> dict:
    """{kernel: (launches, total_ms)} of the launches recorded since the last reset."""
    import json
    need = _lib.fbs_profile_report(None, 0)
    if need < 0:
        _check(-need)
    buf = C.create_string_buffer(need + 16)
    _lib.fbs_profile_report(buf, len(buf))
    return {k: (int(v[0]), float(v[1])) for k, v in json.loads(buf.value.decode()).items()}


# ----------------------------------------------------------------------------- grid
class Grid:
    """Handle of a built simplified bilateral grid (fbs_grid)."""

    def __init__(self, handle, frames, H, W):
        self._h = handle
        self.frames, self.H, self.W = frames, H, W
        self.N = frames * H * W
        self._sizes = None  # (M, levels): data-dependent, read back on first use (one stream sync)

    def _read_sizes(self):
        if self._sizes is None:
            m, lv = _i64(), _i()
            _check(_lib.fbs_grid_info(self._h, None, C.byref(m), C.byref(lv), None, None, None))
            self._sizes = (m.value, lv.value)
        return self._sizes

    @property
    def M(self):
        """Vertices (all frames).  The build is asynchronous: the first query synchronises."""
        return self._read_sizes()[0]

    @property
    def levels(self):
        return self._read_sizes()[1]

    @property
    def handle(self):
        return self._h

    def info(self):
        fv = np.zeros(self.frames, np.int64)
        lv = np.zeros(self.levels, np.int64)
        fl = np.zeros(self.frames, np.int32)
        _check(_lib.fbs_grid_info(self._h, None, None, None, _np_ptr(fv), _np_ptr(lv), _np_ptr(fl)))
        return {"N": self.N, "M": self.M, "levels": self.levels, "frame_vertices": fv,
                "level_vertices": lv, "frame_levels": fl}

    def export(self):
        keys = np.zeros(self.M, np.uint64)
        vid = np.zeros(self.N, np.int32)
        nbr = np.zeros((self.M, 10), np.int32)
        m = np.zeros(self.M, np.int32)
        n = np.zeros(self.M, np.float32)
        res = np.zeros(1, np.float32)
        _check(_lib.fbs_grid_export(self._h, _np_ptr(keys), _np_ptr(vid), _np_ptr(nbr), _np_ptr(m),
                                    _np_ptr(n), _np_ptr(res)))
        return {"keys": keys, "vid": vid, "nbr": nbr, "m": m, "n": n, "bistoch_residual": float(res[0])}

    def pyramid_level(self, level: int):
        lv = self.info()["level_vertices"]
        keys = np.zeros(int(lv[level]), np.uint64)
        parent = np.zeros(int(lv[level - 1]), np.int32)
        count = np.zeros(int(lv[level]), np.int32)
        _check(_lib.fbs_pyramid_export(self._h, level, _np_ptr(keys), _np_ptr(parent), _np_ptr(count)))
        return {"keys": keys, "parent": parent, "count": count}

    def close(self):
        if self._h is not None:
            _lib.fbs_grid_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def grid_build(rgb: torch.Tensor, sigma_xy: float, sigma_l: float, sigma_uv: float, n_bistoch: int = 20,
               build_pyramid: bool = True, stream=None, dims: int = 5) -> Grid:
    """fbs_grid_build: rgb uint8 CUDA [F][H][W][3] (or [H][W][3]); dims = 3 builds the XYL grid
    of a grayscale reference."""
    if isinstance(rgb, torch.Tensor) and rgb.dim() == 3:
        rgb = rgb.unsqueeze(0)
    rgb = _dev_tensor(rgb, torch.uint8, "rgb", 4)
    F, H, W, ch = rgb.shape
    if ch != 3:
        raise ValueError("rgb must be [F][H][W][3]")
    o = GridOpts(int(n_bistoch), int(bool(build_pyramid)), int(dims))
    h = C.c_void_p()
    _check(_lib.fbs_grid_build(_ptr(rgb), F, H, W, float(sigma_xy), float(sigma_l), float(sigma_uv),
                               C.byref(o), _stream(stream), C.byref(h)))
    return Grid(h, F, H, W)


# ----------------------------------------------------------------------------- solve
def make_opts(precond="hier", init="hier", mode="fixed", iters=25, tol=1e-6, max_iters=2000,
              precond_alpha=2.0, precond_beta=5.0, init_alpha=4.0, init_beta=0.0, lowrank_eps=0.0) -> SolveOpts:
    return SolveOpts(PRECOND[precond], INIT[init], MODE[mode], int(iters), float(tol), int(max_iters),
                     float(precond_alpha), float(precond_beta), float(init_alpha), float(init_beta),
                     float(lowrank_eps))


class System:
    """Handle of a solved system (fbs_system): A-state, M⁻¹ and ŷ, reused by backward."""

    def __init__(self, handle, grid: Grid, K: int):
        self._h = handle
        self.grid = grid
        self.K = K

    def stats(self):
        FK = self.grid.frames * self.K
        it = np.zeros(FK, np.int32)
        rel = np.zeros(FK, np.float64)
        bit = np.zeros(FK, np.int32)
        st = np.zeros(1, np.int32)
        _check(_lib.fbs_system_stats(self._h, _np_ptr(it), _np_ptr(rel), _np_ptr(bit), _np_ptr(st)))
        return {"iterations": it.reshape(self.grid.frames, self.K), "relres": rel.reshape(self.grid.frames, self.K),
                "bwd_iterations": bit.reshape(self.grid.frames, self.K), "status": int(st[0])}

    def export(self):
        M, K = self.grid.M, self.K
        sc = np.zeros(M, np.float32)
        b = np.zeros((M, K), np.float32)
        dA = np.zeros(M, np.float32)
        y0 = np.zeros((M, K), np.float32)
        y = np.zeros((M, K), np.float32)
        db = np.zeros((M, K), np.float32)
        _check(_lib.fbs_system_export(self._h, _np_ptr(sc), _np_ptr(b), _np_ptr(dA), _np_ptr(y0), _np_ptr(y),
                                      _np_ptr(db)))
        return {"sc": sc, "b": b, "diagA": dA, "y0": y0, "y": y, "db": db}

    def backward(self, dldx: torch.Tensor, t: torch.Tensor, c: torch.Tensor, stream=None):
        """fbs_solve_backward → (dL/dt [F][K][H][W], dL/dc [F][H][W])."""
        g = self.grid
        dldx = _dev_tensor(dldx, torch.float32, "dldx", 4)
        t = _dev_tensor(t, torch.float32, "t", 4)
        c = _dev_tensor(c, torch.float32, "c", 3)
        dt = torch.empty_like(t)
        dc = torch.empty_like(c)
        _check(_lib.fbs_solve_backward(self._h, _ptr(dldx), _ptr(t), _ptr(c), _ptr(dt), _ptr(dc), _stream(stream)))
        return dt, dc

    def apply_A(self, y: torch.Tensor, stream=None) -> torch.Tensor:
        y = _dev_tensor(y, torch.float32, "y", 2)
        out = torch.empty_like(y)
        _check(_lib.fbs_system_apply_A(self._h, _ptr(y), _ptr(out), _stream(stream)))
        return out

    def apply_precond(self, r: torch.Tensor, stream=None) -> torch.Tensor:
        r = _dev_tensor(r, torch.float32, "r", 2)
        out = torch.empty_like(r)
        _check(_lib.fbs_system_apply_precond(self._h, _ptr(r), _ptr(out), _stream(stream)))
        return out

    def close(self):
        if self._h is not None:
            _lib.fbs_system_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve(grid: Grid, t: torch.Tensor, c: torch.Tensor, lam: float, want_y: bool = False,
          keep_system: bool = False, stream=None, out: Optional[torch.Tensor] = None, **opts):
    """fbs_solve.  t float32 [F][K][H][W], c float32 [F][H][W] → x [F][K][H][W]
    (+ y [M][K] if want_y, + System if keep_system)."""
    t = _dev_tensor(t, torch.float32, "t", 4)
    c = _dev_tensor(c, torch.float32, "c", 3)
    F, K, H, W = t.shape
    if (F, H, W) != (grid.frames, grid.H, grid.W) or tuple(c.shape) != (F, H, W):
        raise ValueError("t/c shapes do not match the grid")
    x = _out_tensor(out, t)
    y = torch.empty((grid.M, K), dtype=torch.float32, device=t.device) if want_y else None
    o = make_opts(**opts)
    h = C.c_void_p()
    _check(_lib.fbs_solve(grid.handle, _ptr(t), K, _ptr(c), float(lam), C.byref(o), _ptr(x), _ptr(y),
                          C.byref(h) if keep_system else None, _stream(stream)))
    res = [x]
    if want_y:
        res.append(y)
    if keep_system:
        res.append(System(h, grid, K))
    return res[0] if len(res) == 1 else tuple(res)


def solve_robust(grid: Grid, t: torch.Tensor, c_init: torch.Tensor, lam: float, sigma_gm: float, n_irls: int,
                 want_weights: bool = False, stream=None, out: Optional[torch.Tensor] = None, **opts):
    """fbs_solve_robust (Supp. Alg. 3): t float32 [F][1][H][W], c_init float32 [F][H][W] →
    x [F][1][H][W] (+ the final IRLS weights [F][H][W] if want_weights)."""
    t = _dev_tensor(t, torch.float32, "t", 4)
    c_init = _dev_tensor(c_init, torch.float32, "c_init", 3)
    F, K, H, W = t.shape
    if (F, H, W) != (grid.frames, grid.H, grid.W) or tuple(c_init.shape) != (F, H, W):
        raise ValueError("t/c_init shapes do not match the grid")
    x = _out_tensor(out, t)
    w = torch.empty_like(c_init) if want_weights else None
    o = make_opts(**opts)
    _check(_lib.fbs_solve_robust(grid.handle, _ptr(t), K, _ptr(c_init), float(lam), C.byref(o), float(sigma_gm),
                                 int(n_irls), _ptr(x), _ptr(w), _stream(stream)))
    return (x, w) if want_weights else x


def dt_filter(rgb: torch.Tensor, x: torch.Tensor, sigma_s: float, sigma_r: float, n_iters: int = 3,
              out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """fbs_dt_filter: domain-transform post-filter of x float32 [F][K][H][W] guided by rgb uint8
    [F][H][W][3] (reading #28)."""
    if isinstance(rgb, torch.Tensor) and rgb.dim() == 3:
        rgb = rgb.unsqueeze(0)
    rgb = _dev_tensor(rgb, torch.uint8, "rgb", 4)
    x = _dev_tensor(x, torch.float32, "x", 4)
    F, K, H, W = x.shape
    if tuple(rgb.shape) != (F, H, W, 3):
        raise ValueError("rgb must be [F][H][W][3] matching x")
    y = _out_tensor(out, x)
    _check(_lib.fbs_dt_filter(_ptr(rgb), F, H, W, _ptr(x), K, float(sigma_s), float(sigma_r), int(n_iters), _ptr(y),
                              _stream(stream)))
    return y


# ----------------------------------------------------------------------------- operators
def slice_(grid: Grid, y: torch.Tensor, stream=None) -> torch.Tensor:
    y = _dev_tensor(y, torch.float32, "y", 2)
    K = y.shape[1]
    x = torch.empty((grid.frames, K, grid.H, grid.W), dtype=torch.float32, device=y.device)
    _check(_lib.fbs_slice(grid.handle, _ptr(y), K, _ptr(x), _stream(stream)))
    return x


def splat(grid: Grid, p: torch.Tensor, stream=None) -> torch.Tensor:
    p = _dev_tensor(p, torch.float32, "p", 4)
    K = p.shape[1]
    out = torch.empty((grid.M, K), dtype=torch.float32, device=p.device)
    _check(_lib.fbs_splat(grid.handle, _ptr(p), K, _ptr(out), _stream(stream)))
    return out


def blur(grid: Grid, v: torch.Tensor, stream=None) -> torch.Tensor:
    v = _dev_tensor(v, torch.float32, "v", 1)
    out = torch.empty_like(v)
    _check(_lib.fbs_blur(grid.handle, _ptr(v), _ptr(out), _stream(stream)))
    return out


# Every (callbacks, Allocator) pair ever registered stays alive for the life of the process:
# handles copy the allocator's function pointers when they are created and call them again when
# destroyed, possibly after the allocator was replaced or disabled.
_torch_alloc_refs = []


def use_torch_allocator(enable: bool = True):
    """Route the device buffers of handles created from now on through PyTorch's caching
    allocator (stream-ordered on the handle's stream); False restores cudaMallocAsync."""
    if not enable:
        _check(_lib.fbs_set_allocator(None))
        return

    def _alloc(nbytes, ctx, stream):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), device=torch.cuda.current_device(),
                                                      stream=int(stream or 0))
        except Exception:  # noqa: BLE001 (the C side reports FBS_ENOMEM)
            return None

    def _free(ptr, ctx, stream):
        torch.cuda.caching_allocator_delete(int(ptr))

    refs = (_ALLOC_FN(_alloc), _FREE_FN(_free))
    a = Allocator(refs[0], refs[1], None)
    _torch_alloc_refs.append((refs, a))
    _check(_lib.fbs_set_allocator(C.byref(a)))


def header_symbols():
    """Function names declared in include/fbs.h (for ABI-completeness tests)."""
    import re
    with open(os.path.join(os.path.dirname(_HERE), "include", "fbs.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(fbs_[a-z_]+)\s*\(", text)))
