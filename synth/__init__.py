"""Seeded synthetic point sets shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the method (no keys, no trees, no distances):
it only draws coordinates. Both `oracle/` and `paper_2604_05885_b200/` consumers
take their inputs from here, which is the one module the two sides share.
"""
from .generators import (  # noqa: F401
    splitmix64,
    uniform_points,
    clustered_points,
    normal_points,
    lattice_points,
    make_config,
    CONFIGS,
)
