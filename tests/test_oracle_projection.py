"""Oracle pins of the projection operators ("apply the pressure
gradient to project the velocity field and measure the divergence"): the algebraic identity
divergence(u - G p) = divergence(u) - A p on random graded trees (flux consistency with the
composite operator, Eq. 11), exact divergence of affine velocity fields, exact gradients of
linear pressures across T-junctions (Eq. 12), and the tank's right-hand side."""
import numpy as np
import pytest

from octgen import canonical_order, sphere_band_tiles, uniform_tiles
from oracle.oracle import Oracle, tank_fields
from tests.helpers import random_graded_tree


def _sorted(t):
    return t[canonical_order(t)]


def _geom(o):
    X, Y, Z, lev = o.cell_coords()
    n = o.N
    h = np.ldexp(1.0, -lev[:n]) / 8
    cen = np.stack([(X[:n] + 0.5) * h, (Y[:n] + 0.5) * h, (Z[:n] + 0.5) * h], axis=1)
    return cen, h


def _face_field(o, fn):
    """per-face values from a function of the face centre: both cells of a shared face see
    the same value (consistent copies, as a geometry pipeline produces them)"""
    cen, h = _geom(o)
    out = np.zeros((6, o.N), dtype=np.float32)
    for f in range(6):
        pc = cen.copy()
        pc[:, f // 2] += (f % 2 - 0.5) * h
        out[f] = fn(pc)
    return out


@pytest.mark.parametrize("seed", range(4))
def test_divergence_of_projection_equals_div_minus_Ap(seed):
    """Random graded trees, smooth random face fractions and betas, random Neumann (solid)
    cells and walls: for random u and p, div(u - G p) = div(u) - A p (the composite fluxes
    are conservative, Eq. 11, and G p is built from the operator's own face fluxes)."""
    rng = np.random.default_rng(seed)
    t = random_graded_tree(rng, 1, 3, 0.35)
    walls = tuple(int(v) for v in rng.integers(0, 2, 6))
    o = Oracle(t, wall_bc=walls)
    kind = np.where(rng.random(o.N) < 0.15, 2, 0).astype(np.uint8)
    k1, k2, k3 = rng.uniform(5, 20, 3)
    frac = _face_field(o, lambda q: 0.05 + 0.95 * (0.5 + 0.5 * np.sin(k1 * q[:, 0] + 3 * q[:, 1]) * np.cos(k2 * q[:, 2])))
    beta = _face_field(o, lambda q: 1.0 + 0.5 * np.sin(k3 * (q[:, 0] + 2 * q[:, 1] + 3 * q[:, 2])))
    o.setup(kind, (frac * beta).astype(np.float32))
    u = rng.standard_normal((6, o.N))
    p = rng.standard_normal(o.N)
    act = o.coefs()[:o.N, 0] != 0
    u2 = o.subtract_gradient(frac, p, u)
    lhs = o.divergence(frac, u2)
    rhs = o.divergence(frac, u) - o.apply(p)
    scale = np.abs(rhs).max()
    assert np.abs(lhs - rhs)[act].max() <= 1e-12 * scale
    assert np.all(lhs[~act] == 0.0)


def test_face_fluxes_sum_to_operator_row():
    rng = np.random.default_rng(3)
    t = _sorted(sphere_band_tiles(2, 2, r=0.3))
    o = Oracle(t)
    o.setup()
    p = rng.standard_normal(o.N)
    Ap = o.apply(p)
    for k in rng.choice(o.N, 50, replace=False):
        F = o.face_fluxes(k // 512, k % 512, p)
        assert F.sum() == pytest.approx(Ap[k], rel=1e-12, abs=1e-14)


def test_divergence_of_affine_field_exact():
    """u = (2x + 1, -3y, 0.5 z + y) sampled at face centres, all fluid: the midpoint flux is
    exact for affine fields, so b_i = -V_i (2 - 3 + 0.5) on every cell of a graded tree,
    coarse cells at T-junctions included (their faces summed from the fine sides)."""
    t = _sorted(sphere_band_tiles(2, 2, r=0.3))
    o = Oracle(t)
    o.setup()
    cen, h = _geom(o)
    u = np.zeros((6, o.N))
    for f in range(6):
        a, side = f // 2, f % 2
        pc = cen.copy()
        pc[:, a] += (side - 0.5) * h
        comp = [2 * pc[:, 0] + 1, -3 * pc[:, 1], 0.5 * pc[:, 2] + pc[:, 1]][a]
        u[f] = comp
    frac = np.ones((6, o.N), dtype=np.float32)
    b = o.divergence(frac, u)
    assert np.allclose(b, -(h ** 3) * (2 - 3 + 0.5), rtol=1e-12, atol=1e-15)


def test_gradient_of_linear_pressure_exact_across_t_junctions():
    """p = 0.7 x - 1.3 y + 0.4 z, all fluid, Neumann walls: every interior face's normal
    velocity changes by exactly -dp/dn, at T-junctions on both sides (Eq. 12 exactness)."""
    t = _sorted(sphere_band_tiles(2, 2, r=0.3))
    o = Oracle(t, wall_bc=(0, 0, 0, 0, 0, 0))
    o.setup()
    cen, h = _geom(o)
    g = np.array([0.7, -1.3, 0.4])
    p = cen @ g
    frac = np.ones((6, o.N), dtype=np.float32)
    u2 = o.subtract_gradient(frac, p, np.zeros((6, o.N)))
    for f in range(6):
        a, side = f // 2, f % 2
        face = cen[:, a] + (side - 0.5) * h
        interior = (face > 1e-12) & (face < 1 - 1e-12)
        assert np.allclose(u2[f][interior], -g[a], rtol=0, atol=1e-12)
        assert np.all(u2[f][~interior] == 0.0)


def test_tank_rhs_is_divergence_of_downward_velocity():
    """The tank scene's b = h^2 (w_y+ - w_y-) is the divergence of u = (0, -1, 0)."""
    t = _sorted(sphere_band_tiles(2, 2, r=0.3))
    kind, w, b = tank_fields(t, radius=0.3)
    o = Oracle(t, wall_bc=(0, 0, 0, 1, 0, 0))
    o.setup(kind, w)
    u = np.zeros((6, o.N))
    u[2] = u[3] = -1.0
    d = o.divergence(w, u)
    act = o.coefs()[:o.N, 0] != 0
    # same-level faces: identical; coarse cells at T-junctions sum the fine faces
    assert np.allclose(d[act], b[act].astype(np.float64), rtol=1e-6, atol=1e-9)
