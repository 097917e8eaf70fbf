"""Seeded synthetic workload generators shared by the oracle side and the CUDA side.

This module holds NONE of the solver's arithmetic (no coefficients, no operator, no
cycle).  It only produces the problem statement the paper's solver consumes
(Sec. 5.1 L1205-1229 grid construction; Sec. 5.4 L1605-1616 tank scene):

* leaf-tile lists ``(level, i, j, k)`` of 8^3-cell tiles,
* per-leaf-cell kinds (fluid / Dirichlet / Neumann),
* per-leaf-cell face weights ``w = beta * fluid_fraction``,
* right-hand sides.

Per-cell arrays are laid out in the library's canonical leaf-slot order
(level descending, Morton ascending within a level, ``x + 8y + 64z`` within a tile),
which is part of the published ABI contract (include/octmg.h); the generator only
needs the ordering, not any solver data.
"""
from .trees import (  # noqa: F401
    morton3, canonical_order, uniform_tiles, octant_tiles, sphere_band_tiles,
    grade_repair, is_graded, leaf_cell_geometry, tile_counts_by_level,
)
from .fields import (  # noqa: F401
    FLUID, DIRICHLET, NEUMANN, splitmix64_uniform, sinusoid_rhs, random_rhs,
    tank_fields, face_fraction_marching_squares,
)
from .configs import make_config, CONFIG_NAMES  # noqa: F401
