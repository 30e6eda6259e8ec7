"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads without a GPU, exports every
symbol include/fbs.h declares, validates arguments, and has no CPU fallback."""
import ctypes
import importlib.util
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1511_03296_b200", "libfbs.so")


def _build():
    spec = importlib.util.spec_from_file_location("fbs_build", os.path.join(ROOT, "paper_1511_03296_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.build()


@pytest.fixture(scope="module")
def lib():
    _build()
    return ctypes.CDLL(LIB)


def header_functions():
    with open(os.path.join(ROOT, "include", "fbs.h")) as fh:
        text = fh.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fbs_[a-z_]+)\s*\(", text)))


def test_exports_every_declared_symbol(lib):
    names = header_functions()
    assert len(names) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (fbs_[a-z_]+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        getattr(lib, n)


def test_sm100a_code_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_argument_validation_without_gpu(lib):
    lib.fbs_grid_build.restype = ctypes.c_int
    h = ctypes.c_void_p()
    rc = lib.fbs_grid_build(None, 1, 4, 4, ctypes.c_double(8.0), ctypes.c_double(4.0), ctypes.c_double(3.0), None,
                            None, ctypes.byref(h))
    assert rc == 1  # FBS_EINVAL (null rgb) before touching the device
    lib.fbs_last_error.restype = ctypes.c_char_p
    assert b"null" in lib.fbs_last_error()
    rc = lib.fbs_solve(None, None, 1, None, ctypes.c_double(1.0), None, None, None, None, None)
    assert rc == 1


def test_no_cpu_fallback(lib):
    """With a (non-null) pointer but no usable GPU, the library fails loudly (FBS_ECUDA)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    buf = ctypes.create_string_buffer(48)
    h = ctypes.c_void_p()
    rc = lib.fbs_grid_build(buf, 1, 4, 4, ctypes.c_double(8.0), ctypes.c_double(4.0), ctypes.c_double(3.0), None,
                            None, ctypes.byref(h))
    assert rc == 3  # FBS_ECUDA


def test_default_opts(lib):
    class SolveOpts(ctypes.Structure):
        _fields_ = [("precond", ctypes.c_int), ("init", ctypes.c_int), ("mode", ctypes.c_int), ("iters", ctypes.c_int),
                    ("tol", ctypes.c_double), ("max_iters", ctypes.c_int), ("precond_alpha", ctypes.c_double),
                    ("precond_beta", ctypes.c_double), ("init_alpha", ctypes.c_double), ("init_beta", ctypes.c_double),
                    ("lowrank_eps", ctypes.c_double)]
    o = SolveOpts()
    lib.fbs_default_solve_opts(ctypes.byref(o))
    # PAPER.md:285 (α=2, β=5), :293 (α=4, β=0), :334 (25 iterations); low-rank reduction off
    assert (o.precond_alpha, o.precond_beta, o.init_alpha, o.init_beta, o.iters) == (2.0, 5.0, 4.0, 0.0, 25)
    assert o.lowrank_eps == 0.0
    # the binding's struct has the same layout as the header's
    import paper_1511_03296_b200.fbs as F
    assert ctypes.sizeof(F.SolveOpts) == ctypes.sizeof(SolveOpts)


def test_oracle_is_not_imported_by_product():
    """The product package never imports oracle/ (DESIGN.md §2)."""
    pkg = os.path.join(ROOT, "paper_1511_03296_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                with open(os.path.join(dirpath, f), errors="ignore") as fh:
                    src = fh.read()
                assert "oracle" not in re.findall(r"(?:import|from)\s+(oracle)\b", src), f
