"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA path.

This package holds *input recipes only*: grids, masks, initial magnetisations,
B_rms maps and the per-config physical parameters of BASELINE.json configs[0..4]
(SURVEY.md §8(d)).  It contains none of the method's arithmetic (no field, no
torque, no integrator, no cavity recursion) and imports neither ``oracle`` nor
``paper_2410_00966_b200``.
"""
from .configs import (  # noqa: F401
    Config, CONFIGS, make_config, small_config,
    sphere_mask, disc_mask, random_unit, tilted_uniform, vortex_state,
    two_wire_map, strip_map, uniform_brms_for_g,
)
