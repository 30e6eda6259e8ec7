"""Seeded synthetic workloads for the bilateral-space solve.

This module holds NO arithmetic of the method (no colour transform, no
quantisation, no splat/blur/solve).  It only draws reference images, targets,
confidences and upstream gradients from seeded NumPy generators, with the
shapes and value structure of BASELINE.json's configs.  Both the oracle tests
and the CUDA path consume it; neither depends on the other.
"""
from .synth import (  # noqa: F401
    Workload,
    CONFIGS,
    make,
    voronoi_reference,
    planar_depth,
)
