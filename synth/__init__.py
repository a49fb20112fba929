"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no window, no psi-hat, no FFT, no
gather).  It only draws nodes x_j and spectra f^(k) with the shapes and value
distributions of BASELINE.json's configs (recipe: SURVEY.md §8(d), restated in
DESIGN.md "Input recipe").  Both `oracle/` and the GPU tests/bench consume the
identical arrays produced here.
"""
from .inputs import (  # noqa: F401
    CONFIGS,
    Config,
    SEED_BASE,
    make_nodes,
    make_spectrum,
    feasible_box_nodes,
    grid_point_nodes,
    triangle_spectrum,
    ones_spectrum,
    chebyshev_nodes,
)
