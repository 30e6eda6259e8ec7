"""B200-native bilateral-space solve (Fast Bilateral Solver, arXiv 1511.03296).

The product is libfbs.so (C ABI: include/fbs.h, sm_100a kernels in csrc/); this package
is its thin ctypes binding.  Importing it fails loudly if the library is missing.
"""
from .fbs import (  # noqa: F401
    FbsError,
    Grid,
    System,
    blur,
    dt_filter,
    grid_build,
    launch_count,
    make_opts,
    profile_enable,
    profile_report,
    profile_reset,
    slice_,
    solve,
    solve_robust,
    use_torch_allocator,
    splat,
    version,
)
