"""Oracle pins of the GMG comparison mode: the cycle's coarse records "given
directly by the grid discretization" — Eq. 3 assembled on every inner cell from its
own kind and face weights — instead of Alg. 3.

* fluid-only systems: equal to the Galerkin (Alg. 3) records ("in fluid-only
  systems, the matrix given by the Galerkin principle is equivalent to the matrix given
  directly by the grid discretization"), on adaptive trees and with random face weights;
* next to a solid cell: the closed forms 6 h_c (grid) vs 21/4 h_c (Galerkin: "the
  terms related to i will vanish from A_II^{l-1}");
* the composite operator the PCG solves is unchanged; the GMG cycle is linear, and a symmetric
  preconditioner on a uniform tree with an obstacle;
* on the cut-cell tank the GMG-preconditioned PCG needs clearly more iterations than the
  algebraically consistent cycle (Fig. 12)."""
import numpy as np
import pytest

from octgen import canonical_order, make_config, sphere_band_tiles, uniform_tiles
from oracle.oracle import Oracle, tank_fields
from tests.helpers import random_graded_tree


def _sorted(t):
    return t[canonical_order(t)]


def _children_mean_weights(o, w_leaf):
    """Inner-cell face weights = the mean of the four child sub-face weights of each face
    (children first, bottom-up), i.e. the coarse face's fluid area fraction."""
    X, Y, Z, lev = o.cell_coords()
    NL3 = o.NL * o.B3
    idx = {(int(l), int(x), int(y), int(z)): n for n, (l, x, y, z) in enumerate(zip(lev, X, Y, Z))}
    w_all = np.zeros((6, o.T * o.B3))
    w_all[:, :NL3] = w_leaf
    order = np.argsort(-lev[NL3:], kind="stable") + NL3  # finest inner level first
    for n in order:
        l, x, y, z = int(lev[n]), int(X[n]), int(Y[n]), int(Z[n])
        for f in range(6):
            a, s = f // 2, f & 1
            acc = 0.0
            for d in range(8):
                dd = (d & 1, (d >> 1) & 1, d >> 2)
                if dd[a] != s:
                    continue
                acc += w_all[f, idx[(l + 1, 2 * x + dd[0], 2 * y + dd[1], 2 * z + dd[2])]]
            w_all[f, n] = acc / 4.0
    return w_all[:, NL3:].astype(np.float32)


@pytest.mark.parametrize("seed", range(4))
def test_gmg_equals_galerkin_on_fluid_only_adaptive_trees(seed):
    rng = np.random.default_rng(seed)
    tiles = random_graded_tree(rng, l0=1, lmax=3, p_refine=0.35) if seed else _sorted(sphere_band_tiles(2, 2, r=0.25))
    walls = tuple(int(v) for v in rng.integers(0, 2, 6)) if seed else (1, 1, 1, 1, 1, 1)
    o = Oracle(tiles, wall_bc=walls, B=4)
    o.setup()
    g = o.coefs()
    o.setup_gmg()
    c = o.coefs_cycle()
    assert np.array_equal(o.coefs(), g)  # the composite operator's records are untouched
    scale = np.abs(g).max()
    assert np.abs(c - g).max() <= 1e-12 * scale


@pytest.mark.parametrize("seed", range(3))
def test_gmg_equals_galerkin_with_random_weights_uniform_tree(seed):
    """Random face weights on a uniform tree: the grid records with every coarse face weight the
    mean of its four sub-face weights equal Alg. 3's (no T-junction faces)."""
    rng = np.random.default_rng(10 + seed)
    o = Oracle(_sorted(uniform_tiles(2)), wall_bc=tuple(int(v) for v in rng.integers(0, 2, 6)), B=4)
    w = rng.uniform(0.2, 1.0, (6, o.N)).astype(np.float32)
    o.setup(None, w)
    g = o.coefs()
    o.setup_gmg(None, _children_mean_weights(o, w))
    assert np.abs(o.coefs_cycle() - g).max() <= 1e-6 * np.abs(g).max()  # fp32 weight means


def test_gmg_closed_form_next_to_a_solid_child():
    """One solid (Neumann) leaf cell at a block corner, all else fluid, w = 1: its parent's grid
    record is Eq. 3's 6 h_c / -h_c; Alg. 3 gives (3 * 5 + 4 * 6 - 2 * 9) h_f / 2 = 21/4 h_c."""
    o = Oracle(_sorted(uniform_tiles(1)))  # 16^3 leaves, 8^3 level-0 cells
    kind = np.zeros(o.N, dtype=np.uint8)
    X, Y, Z, lev = o.cell_coords()
    leaf = np.flatnonzero((lev == 1) & (X == 6) & (Y == 6) & (Z == 6))[0]
    kind[leaf] = 2
    o.setup(kind)
    par = np.flatnonzero((lev == 0) & (X == 3) & (Y == 3) & (Z == 3))[0]
    hc = 1.0 / 8
    assert np.isclose(o.coefs()[par, 0], 21.0 / 4.0 * hc, rtol=0, atol=1e-15)
    o.setup_gmg()
    cc = o.coefs_cycle()
    assert np.isclose(cc[par, 0], 6 * hc, rtol=0, atol=1e-15)
    assert np.allclose(cc[par, 1:], -hc, rtol=0, atol=1e-15)
    # a solid inner cell (its own kind Neumann) is inactive with a zero record
    ki = np.zeros(o.NI * o.B3, dtype=np.uint8)
    ki[par - o.NL * o.B3] = 2
    o.setup_gmg(ki)
    cc = o.coefs_cycle()
    assert np.all(cc[par] == 0.0)


def test_gmg_cycle_linear_and_operator_unchanged():
    cfg = make_config("tank_small")
    o = Oracle(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
    o.setup(cfg["kind"], cfg["w"])
    rng = np.random.default_rng(5)
    x = np.where(cfg["kind"] == 0, rng.standard_normal(o.N), 0.0)
    y0 = o.apply(x)
    ki, wi, _ = tank_fields(o.tables()["tiles"][o.NL:], cfg["ext"], radius=cfg["radius"])
    o.setup_gmg(ki, wi)
    assert np.array_equal(o.apply(x), y0)
    act = o.coefs_diag_leaf() != 0
    b1 = np.where(act, rng.standard_normal(o.N), 0.0)
    b2 = np.where(act, rng.standard_normal(o.N), 0.0)
    for mu in (1, 2):
        m1, m2 = o.vcycle(b1, mu=mu), o.vcycle(b2, mu=mu)
        assert np.abs(o.vcycle(2.0 * b1 - 3.0 * b2, mu=mu) - (2.0 * m1 - 3.0 * m2)).max() <= 1e-10 * np.abs(m1).max()


def test_gmg_cycle_symmetric_on_uniform_tree_with_obstacle():
    """Uniform tree (no T-junctions), the tank obstacle: the grid-assembled coarse operators have
    one coupling per face, so the RB / BR-symmetric cycle stays a symmetric preconditioner."""
    t = _sorted(uniform_tiles(2))
    o = Oracle(t, wall_bc=(0, 0, 0, 1, 0, 0), B=4)
    kind, w, _ = tank_fields(t, radius=0.3, B=4)
    o.setup(kind, w)
    ki, wi, _ = tank_fields(o.tables()["tiles"][o.NL:], radius=0.3, B=4)
    o.setup_gmg(ki, wi)
    assert np.abs(o.coefs_cycle() - o.coefs()).max() > 1e-3 * np.abs(o.coefs()).max()  # not Galerkin here
    rng = np.random.default_rng(6)
    act = o.coefs_diag_leaf() != 0
    for mu in (1, 2):
        b1 = np.where(act, rng.standard_normal(o.N), 0.0)
        b2 = np.where(act, rng.standard_normal(o.N), 0.0)
        a, c = o.vcycle(b1, mu=mu) @ b2, b1 @ o.vcycle(b2, mu=mu)
        assert abs(a - c) <= 1e-10 * abs(a)


def test_gmg_slower_than_algebraic_coarsening_on_cut_cells():
    """Fig. 12: on the cut-cell tank the GMG preconditioner 'fails to converge
    effectively' while the algebraically consistent W-cycle converges fastest."""
    cfg = make_config("tank_small")
    o = Oracle(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
    o.setup(cfg["kind"], cfg["w"])
    b = cfg["b"].astype(np.float64)
    ours = o.pcg(b, rtol=1e-6, mu=2, max_iters=100)
    ki, wi, _ = tank_fields(o.tables()["tiles"][o.NL:], cfg["ext"], radius=cfg["radius"])
    o.setup_gmg(ki, wi)
    gmg = o.pcg(b, rtol=1e-6, mu=2, max_iters=100)
    assert ours["status"] == "OK" and gmg["status"] == "OK"
    assert gmg["iters"] >= ours["iters"] + 4, (ours["iters"], gmg["iters"])
    assert gmg["history"][1] > 10 * ours["history"][1]
