"""Oracle pins of the cycle variants: literal Alg. 3 (P:L480-525 as printed,
DESIGN.md reading 3) and multigrid as a standalone solver."""
import numpy as np
import pytest

from octgen import canonical_order, make_config, uniform_tiles
from octgen.fields import sinusoid_rhs
from oracle.oracle import Oracle
from tests.helpers import dense_composite, random_graded_tree


def _sorted(t):
    return t[canonical_order(t)]


@pytest.mark.parametrize("seed", range(4))
def test_literal_alg3_equals_activity_tested_without_dirichlet_cells(seed):
    """With no Dirichlet cell, a nonzero stored -face coupling c_{i,e-} implies both sides are
    active fluid, so the bracketed activity test of reading 3 never fires: literal Alg. 3 and
    the activity-tested Alg. 3 give identical hierarchies (random Neumann masks and weights on
    random graded trees, Dirichlet and Neumann walls)."""
    rng = np.random.default_rng(seed)
    t = random_graded_tree(rng, 1, 3, 0.3)
    walls = tuple(int(v) for v in rng.integers(0, 2, 6))
    o1, o2 = Oracle(t, wall_bc=walls), Oracle(t, wall_bc=walls)
    kind = np.where(rng.random(o1.N) < 0.2, 2, 0).astype(np.uint8)
    w = rng.random((6, o1.N)).astype(np.float32)
    o1.setup(kind, w)
    o2.setup(kind, w, coarsen_literal=True)
    assert np.array_equal(o1.coefs(), o2.coefs())


def test_literal_alg3_keeps_dirichlet_cross_term_closed_form():
    """16^3 uniform (level-1 tiles), all fluid, w = 1, one Dirichlet cell at X=1, Y=Z=4.  The
    coarse cell I = (1, 2, 2) has the four d_x = 0 children X = 2, Y,Z in {4,5}, each with
    c_{i,x-} = -h (P:L328-330 keeps the Dirichlet cross term).  Literal Alg. 3 sums all four:
    c_{I,x-} = 4 (-h)/2 = -2h; the activity test drops the child whose x- neighbour is the
    Dirichlet cell: 3 (-h)/2 = -1.5h (h = 1/16)."""
    t = _sorted(uniform_tiles(1))
    o = Oracle(t)
    kind = np.zeros(o.N, dtype=np.uint8)
    X, Y, Z, lev = o.cell_coords()
    i_d = np.flatnonzero((X[:o.N] == 1) & (Y[:o.N] == 4) & (Z[:o.N] == 4))[0]
    kind[i_d] = 1
    h = 1.0 / 16
    I = np.flatnonzero((lev == 0) & (X == 1) & (Y == 2) & (Z == 2))[0]
    o.setup(kind)
    assert o.coefs()[I, 1] == pytest.approx(-1.5 * h, abs=1e-15)
    o.setup(kind, coarsen_literal=True)
    cf = o.coefs()
    assert cf[I, 1] == pytest.approx(-2.0 * h, abs=1e-15)
    # the y-/z- couplings of I and its diagonal are untouched by the literal reading
    o2 = Oracle(t)
    o2.setup(kind)
    assert np.array_equal(cf[I, [0, 2, 3]], o2.coefs()[I, [0, 2, 3]])


@pytest.mark.parametrize("seed", range(3))
def test_standalone_mg_converges_to_dense_solution(seed):
    """x_{k+1} = x_k + M(b - A x_k) with beta = 1 reaches numpy's dense solve on random
    graded B=4 trees with random Dirichlet masks and weights (V- and W-cycle)."""
    rng = np.random.default_rng(100 + seed)
    t = random_graded_tree(rng, 1, 2, 0.4)
    o = Oracle(t, B=4)
    kind = rng.choice([0, 1], size=o.N, p=[0.9, 0.1]).astype(np.uint8)
    w = (0.2 + 0.8 * rng.random((6, o.N))).astype(np.float32)
    o.setup(kind, w)
    act = o.coefs()[:o.N, 0] != 0
    A = dense_composite(o)[np.ix_(act, act)]
    b = rng.standard_normal(o.N) * act
    x_ref = np.zeros(o.N)
    x_ref[act] = np.linalg.solve(A, b[act])
    for mu in (1, 2):
        r = o.mg_solve(b, rtol=1e-11, mu=mu, beta=1.0, max_iters=400)
        assert r["status"] == "OK"
        assert np.linalg.norm(r["x"] - x_ref) <= 1e-10 * np.linalg.cond(A) * np.linalg.norm(x_ref)


def test_standalone_mg_beta1_contracts_every_iteration():
    """With beta = 1 the standalone cycle is a convergent stationary iteration: on the
    Dirichlet sinusoid (16^3, 32^3) the residual falls at every iteration, for the V- and the
    W-cycle.  (The paper gives no standalone rates; with piecewise-constant transfers the
    factor is slow, 0.5-0.8, and grows with the grid, so only contraction is pinned.)"""
    for lev in (1, 2):
        t = _sorted(uniform_tiles(lev))
        o = Oracle(t)
        o.setup()
        b = sinusoid_rhs(t).astype(np.float64)
        for mu in (1, 2):
            r = o.mg_solve(b, rtol=1e-6, beta=1.0, mu=mu, max_iters=200)
            h = np.concatenate([[1.0], r["history"]])
            assert r["status"] == "OK"
            assert np.all(np.diff(h) < 0)
            assert (h[-1] / h[1]) ** (1.0 / (len(h) - 2)) < 0.9


def test_standalone_mg_first_iterate_is_one_cycle():
    """x_1 = M(b) (x_0 = 0): the first iterate of the standalone solver is one cycle of b."""
    cfg = make_config("sphere_small_dir")
    o = Oracle(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
    o.setup(cfg["kind"], cfg["w"])
    b = cfg["b"].astype(np.float64)
    r = o.mg_solve(b, rtol=1e-30, beta=1.0, max_iters=1)
    assert r["status"] == "MAXITER" and r["iters"] == 1
    z = o.vcycle(b, beta=1.0)
    assert np.array_equal(r["x"], z)
