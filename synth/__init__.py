"""Seeded synthetic inputs shared by the oracle (tests) and the CUDA path (bench).

Holds none of the FDK method's arithmetic: only the workload recipe (the five
BASELINE.json configs' scanner geometry), the
ellipsoid phantom table and its analytic line integrals (the paper's
Shepp-Logan methodology), and a counter-based noise field.
"""
from .synth import (  # noqa: F401
    CONFIGS,
    PHANTOM_TABLE,
    ConfigSpec,
    add_noise,
    build,
    config,
    default_ellipsoids,
    density,
    ellipsoids,
    phantom_volume,
    project,
    project_gpu,
    voxel_world,
)
