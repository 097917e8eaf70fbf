"""Oracle pins of the cut-cell geometry (P:L1924 corner SDF samples; SPEC
S:L121-138 marching squares): exact face fractions of planar cuts (linear interpolation is
exact for a linear SDF), the saddle rule, the obstacle-free tank in closed form, and the
sphere's volume / cross-section areas converging to the continuum values."""
import numpy as np
import pytest

from octgen import canonical_order, uniform_tiles, sphere_band_tiles
from oracle.oracle import face_fraction, tank_fields


def _sorted(t):
    return t[canonical_order(t)]


CORNERS = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], dtype=np.float64)


def _plane(a, b, d):
    """corner samples and face-centre sample of phi(x, y) = a x + b y - d on the unit face"""
    phi = a * CORNERS[:, 0] + b * CORNERS[:, 1] - d
    return phi, a * 0.5 + b * 0.5 - d


@pytest.mark.parametrize("a,b,d,expect", [
    (1.0, 0.0, 0.3, 0.7),        # fluid x >= 0.3: rectangle 0.7
    (0.0, -1.0, -0.25, 0.25),    # fluid y <= 0.25
    (1.0, 1.0, 0.5, 0.875),      # solid corner triangle of area 1/8
    (1.0, 1.0, 1.5, 0.125),      # fluid corner triangle of area 1/8
    (2.0, 1.0, 1.0, 0.75),       # trapezoid: solid part (0..0.5 at y=0, 0 at y=1) area 1/4
    (1.0, 0.0, -1.0, 1.0),       # uncut fluid
    (1.0, 0.0, 2.0, 0.0),        # uncut solid
])
def test_planar_cut_fractions_exact(a, b, d, expect):
    phi, pc = _plane(a, b, d)
    assert face_fraction(phi, pc) == pytest.approx(expect, abs=1e-15)


def test_saddle_rule():
    """Diagonal corners alike: a fluid centre joins the fluid corners (1 - two solid
    triangles), a solid centre separates them (two fluid triangles); legs of 1/2 here."""
    phi = np.array([1.0, -1.0, 1.0, -1.0])
    assert face_fraction(phi, +0.5) == pytest.approx(1.0 - 2 * 0.125, abs=1e-15)
    assert face_fraction(phi, -0.5) == pytest.approx(2 * 0.125, abs=1e-15)


def test_obstacle_free_tank_closed_form():
    """No obstacle: all fluid; interior faces w = 1, walls 0 except the open top (w = 1);
    b = h^2 (w_y+ - w_y-) is h^2 on the bottom cell row and 0 elsewhere."""
    t = _sorted(uniform_tiles(1))
    kind, w, b = tank_fields(t, radius=0.0)
    h = 1.0 / 16
    assert np.all(kind == 0)
    off = np.arange(512)
    X = (t[:, 1:2] * 8 + off % 8).ravel()
    Y = (t[:, 2:3] * 8 + (off // 8) % 8).ravel()
    Z = (t[:, 3:4] * 8 + off // 64).ravel()
    for f, (P, lo, wall_w) in enumerate([(X, 0, 0), (X, 15, 0), (Y, 0, 0), (Y, 15, 1), (Z, 0, 0), (Z, 15, 0)]):
        at = P == lo
        assert np.all(w[f][at] == wall_w) and np.all(w[f][~at] == 1.0)
    assert np.allclose(b, np.where(Y == 0, h * h, 0.0), rtol=0, atol=1e-12)


def test_sphere_volume_and_cross_sections():
    """Solid (Neumann) cell volume -> 4/3 pi r^3; the solid part of the x-faces in the plane
    x = 1/2 -> the disc area pi r^2 (marching-squares polygon of the circle)."""
    r, c = 0.3, (0.5, 0.5, 0.5)
    t = _sorted(uniform_tiles(3))  # 64^3
    kind, w, b = tank_fields(t, centre=c, radius=r)
    h = 1.0 / 64
    vol = (kind == 2).sum() * h ** 3
    assert vol == pytest.approx(4.0 / 3.0 * np.pi * r ** 3, rel=0.01)
    off = np.arange(512)
    X = (t[:, 1:2] * 8 + off % 8).ravel()
    at = X == 31  # x+ faces of these cells lie in the plane x = 32 h = 1/2
    solid_area = ((1.0 - w[1][at]) * h * h).sum()
    assert solid_area == pytest.approx(np.pi * r ** 2, rel=2e-3)
    # fluid cells only carry a right-hand side
    assert np.all(b[kind == 2] == 0.0)


def test_adaptive_band_faces_agree_across_levels():
    """On a graded sphere-band tree a face's fraction depends only on the face: the x+ face
    of a fine cell inside the tile equals the x- face of its x+ neighbour (same corners)."""
    t = _sorted(sphere_band_tiles(2, 2, r=0.3))
    kind, w, b = tank_fields(t, radius=0.3)
    n = len(t)
    wx_p = w[1].reshape(n, 8, 8, 8)  # [tile, z, y, x]
    wx_m = w[0].reshape(n, 8, 8, 8)
    assert np.array_equal(wx_p[:, :, :, :7], wx_m[:, :, :, 1:])
