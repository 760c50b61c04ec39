"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no Laplacian, reaction, Euler
update, stamp or probe): only counter-based random numbers, integer geometry
descriptions and phi maps, i.e. the inputs both sides are fed (DESIGN.md §4,
"input recipe"). Shapes are plain dicts that each side converts to its own
struct; membership of a shape is computed by each side independently.
"""
from .gen import splitmix64, stream, noise_plane, half_discs, obstacles  # noqa: F401
from .geometry import and_gate, diode, phi_from_rects  # noqa: F401
from .workloads import PRESET_PX, Workload, barrier, config, preset_cells, spiral_seed  # noqa: F401

PHI_ACTIVE = 0.054   # Table 1
PHI_PASSIVE = 0.0975  # Table 1
