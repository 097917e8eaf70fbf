"""Named workloads (BASELINE.json configs + small parity cases).  Recipe in DESIGN.md.

Boundary setups:
* ``dirichlet``: Dirichlet walls (p = 0 at the virtual wall-cell centre), all cells fluid,
  BC-folded sinusoid RHS (SURVEY c-9; BASELINE config 1 "Dirichlet walls").
* ``neumann_layer``: the paper's Sec. 5.3 sinusoidal test exactly as Table 1 was measured
  (P:L1343 outermost cell layer Neumann, pure-Neumann system, null-space projection
  P:L343), RHS b = V * (-lap f) on fluid cells.
* ``tank``: Sec. 5.4 cut-cell projection (Neumann sides/bottom, Dirichlet top, sphere
  obstacle, b = h^2 (w_y+ - w_y-)).
"""
from __future__ import annotations

import numpy as np

from .trees import canonical_order, uniform_tiles, octant_tiles, sphere_band_tiles
from .fields import (sinusoid_rhs, random_rhs, tank_fields, neumann_layer_kind, NEUMANN)

DIRICHLET_WALLS = (1, 1, 1, 1, 1, 1)
NEUMANN_WALLS = (0, 0, 0, 0, 0, 0)
TANK_WALLS = (0, 0, 0, 1, 0, 0)  # x-,x+,y-,y+,z-,z+ : Neumann sides/bottom, Dirichlet top

# name -> (tile generator, boundary setup, mu, tank obstacle radius)
_TABLE = {
    "cfg1_octant": (lambda: octant_tiles(1), "dirichlet", 1, None),
    "cfg2_uniform256": (lambda: uniform_tiles(5), "neumann_layer", 1, None),
    "cfg3_sphere": (lambda: sphere_band_tiles(4, 3, r=0.375), "neumann_layer", 1, None),
    "cfg4_tank": (lambda: sphere_band_tiles(4, 4, r=0.30), "tank", 2, 0.30),
    "cfg5_tank": (lambda: sphere_band_tiles(4, 5, r=0.35), "tank", 2, 0.35),
    "uniform32": (lambda: uniform_tiles(2), "neumann_layer", 1, None),
    "uniform64": (lambda: uniform_tiles(3), "neumann_layer", 1, None),
    "uniform128": (lambda: uniform_tiles(4), "neumann_layer", 1, None),
    "uniform64_dir": (lambda: uniform_tiles(3), "dirichlet", 1, None),
    "sphere_small": (lambda: sphere_band_tiles(2, 2, r=0.25), "neumann_layer", 1, None),
    "sphere_35": (lambda: sphere_band_tiles(3, 2, r=0.25), "neumann_layer", 1, None),
    "sphere_small_dir": (lambda: sphere_band_tiles(2, 2, r=0.25), "dirichlet", 1, None),
    "tank_small": (lambda: sphere_band_tiles(2, 2, r=0.30), "tank", 2, 0.30),
    "tank_mid": (lambda: sphere_band_tiles(3, 2, r=0.30), "tank", 2, 0.30),
}
CONFIG_NAMES = list(_TABLE)


def make_config(name: str, rhs: str = "default", seed: int = 0, with_fields: bool = True):
    """Returns dict: tiles (canonical leaf order), ext, wall_bc, mu, kind u8[N], w (6,N) f32
    or None, b f32[N].  rhs: 'default' (the setup's analytic RHS) or 'random' (splitmix64
    U(-1,1), zeroed on non-fluid cells)."""
    gen, bc, mu, radius = _TABLE[name]
    tiles = gen()
    tiles = tiles[canonical_order(tiles)]
    walls = {"dirichlet": DIRICHLET_WALLS, "neumann_layer": NEUMANN_WALLS, "tank": TANK_WALLS}[bc]
    cfg = dict(name=name, tiles=tiles, ext=(1, 1, 1), wall_bc=walls, mu=mu, bc=bc, radius=radius,
               n_cells=len(tiles) * 512, kind=None, w=None, b=None)
    if not with_fields:
        return cfg
    N = cfg["n_cells"]
    if bc == "tank":
        kind, w, b = tank_fields(tiles, radius=radius)
    elif bc == "neumann_layer":
        kind = neumann_layer_kind(tiles)
        b = sinusoid_rhs(tiles, wall_bc=NEUMANN_WALLS)
        b[kind == NEUMANN] = 0.0
        w = None
    else:
        kind = np.zeros(N, dtype=np.uint8)
        b = sinusoid_rhs(tiles, wall_bc=DIRICHLET_WALLS)
        w = None
    if rhs == "random":
        b = random_rhs(N, seed)
        b[kind != 0] = 0.0
    cfg.update(kind=kind, w=w, b=b)
    return cfg
