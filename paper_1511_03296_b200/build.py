"""Build libfbs.so (the C-ABI library of include/fbs.h) in-tree for sm_100a.

    python paper_1511_03296_b200/build.py [--force]

One nvcc invocation (unity build of csrc/api.cu), cudart linked statically so the
library loads on hosts without a GPU (every compute call then returns FBS_ECUDA).
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libfbs.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2", "-shared", "-cudart", "static",
    "-Xptxas", "-v",
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build libfbs.so")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(INCLUDE, "fbs.h")])


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False, out: str = None) -> str:
    """Compile csrc/api.cu into `out` (default libfbs.so)."""
    target = out or LIB
    if not force and out is None and not stale():
        return LIB
    extra = os.environ.get("FBS_NVCC_DEFS", "").split()  # A/B builds: e.g. "-DFBS_SP_CHUNK=512"
    cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-I", INCLUDE, os.path.join(CSRC, "api.cu"), "-o", target + ".tmp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    os.replace(target + ".tmp", target)
    if out is None:
        with open(os.path.join(HERE, "ptxas_info.txt"), "w") as fh:
            fh.write(res.stderr)
    if verbose:
        print(res.stderr, file=sys.stderr)
    return target


if __name__ == "__main__":
    # build.py [--force] [-v] [--out PATH]   (--out: an alternative build for FBS_LIB A/B runs)
    o = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, out=o))
