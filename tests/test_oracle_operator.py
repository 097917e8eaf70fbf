"""Oracle composite-operator pins: T-junction flux conservation (Eq. 11),
ghost value (Eq. 12), exactness on affine fields, the tank's exact discrete
solution, the discrete Dirichlet eigenfunction, and the constant null space."""
import numpy as np
import pytest

from octgen import canonical_order, octant_tiles, sphere_band_tiles, uniform_tiles
from octgen.fields import tank_fields
from oracle.oracle import Oracle
from tests.helpers import random_graded_tree

NEU = (0, 0, 0, 0, 0, 0)


def _sorted(t):
    return t[canonical_order(t)]


@pytest.mark.parametrize("seed", range(4))
def test_flux_conservation_pure_neumann(seed):
    """Pure Neumann walls, random face weights w and random x: sum_i (A x)_i = 0, i.e. every
    T-junction face group's fine fluxes equal the coarse flux (Eq. 11), and A 1 = 0."""
    rng = np.random.default_rng(seed)
    t = random_graded_tree(rng, 1, 3, 0.35)
    o = Oracle(t, wall_bc=NEU)
    w = rng.random((6, o.N)).astype(np.float32)
    o.setup(None, w)
    x = rng.standard_normal(o.N)
    y = o.apply(x)
    assert abs(y.sum()) <= 1e-13 * np.abs(y).sum()
    one = o.apply(np.ones(o.N))
    assert np.abs(one).max() <= 1e-15


def test_ghost_worked_example():
    """SPEC S:L155 / Eq. 12: p_f = 1, its siblings 1, coarse p_c = 3 -> g = 2.  With all
    values 1 except the coarse leaf, the fine row changes by -kappa * (g - 1)."""
    t = _sorted(octant_tiles(1))
    o = Oracle(t, wall_bc=NEU)
    o.setup()
    X, Y, Z, lev = o.cell_coords()
    n = o.N
    # fine cell at level 2, X = 15 (the +x face of the refined octant); its +x ghost lies
    # in the level-1 leaf cell (8, Y>>1, Z>>1)
    f = np.where((lev[:n] == 2) & (X[:n] == 15) & (Y[:n] == 3) & (Z[:n] == 5))[0][0]
    cidx = np.where((lev[:n] == 1) & (X[:n] == 8) & (Y[:n] == 1) & (Z[:n] == 2))[0][0]
    x1 = np.ones(n)
    x3 = x1.copy()
    x3[cidx] = 3.0
    kappa = 1.0 / 32  # w = 1, h_f = 1/32
    d = o.apply(x3)[f] - o.apply(x1)[f]
    g_minus_1 = -d / kappa
    assert g_minus_1 == pytest.approx(1.0, rel=1e-14)   # g = 2


@pytest.mark.parametrize("seed", range(3))
def test_affine_exactness_on_graded_tree(seed):
    """All-fluid adaptive tree: for affine u, (A u)_i = 0 at every leaf whose stencil does
    not touch the wall (mean of children and Eq. 12 ghost are exact for affine fields)."""
    rng = np.random.default_rng(10 + seed)
    t = random_graded_tree(rng, 1, 3, 0.35)
    o = Oracle(t, wall_bc=NEU)
    o.setup()
    cen, h = o.leaf_centres()
    a = rng.standard_normal(3)
    u = cen @ a + 0.7
    y = o.apply(u)
    interior = np.all((cen - 1.5 * h[:, None] > 0) & (cen + 1.5 * h[:, None] < 1), axis=1)
    scale = np.abs(a).sum() * h.max() ** 2
    assert np.abs(y[interior]).max() <= 1e-12 * scale


def test_tank_exact_discrete_solution():
    """Obstacle-free tank (Neumann sides/bottom, Dirichlet top, b = h^2 (w_y+ - w_y-)):
    p = 1 + h_top/2 - y solves A p = b exactly on a graded tree (SURVEY c-9)."""
    t = _sorted(sphere_band_tiles(2, 2, center=(0.5, 0.4, 0.5), r=0.2))
    o = Oracle(t, wall_bc=(0, 0, 0, 1, 0, 0))
    kind, w, b = tank_fields(t, radius=0.0)
    o.setup(kind, w)
    cen, h = o.leaf_centres()
    top = cen[:, 1] + 0.5 * h >= 1.0
    h_top = h[top].max()
    assert np.all(h[top] == h_top)
    p = 1.0 + 0.5 * h_top - cen[:, 1]
    r = o.apply(p) - b.astype(np.float64)
    assert np.abs(r).max() <= 1e-12 * np.abs(b).max()


def test_discrete_dirichlet_eigenfunction():
    """Uniform N^3, Dirichlet walls at distance h: u = prod sin(pi (i+1)/(N+1)) satisfies
    A u = 6h (1 - cos(pi/(N+1))) u."""
    t = _sorted(uniform_tiles(2))
    o = Oracle(t)
    o.setup()
    X, Y, Z, _ = o.cell_coords()
    N = 32
    h = 1.0 / N
    s = lambda i: np.sin(np.pi * (i + 1) / (N + 1))
    u = (s(X) * s(Y) * s(Z))[:o.N]
    lam = 6 * h * (1 - np.cos(np.pi / (N + 1)))
    assert np.abs(o.apply(u) - lam * u).max() <= 1e-14
