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


# ---------------------------------------------------------------------------------------
# direct coarsest solve (Alg. 4 line 4, "Or direct solve"; DESIGN reading 9b)
# ---------------------------------------------------------------------------------------
def _level0(o):
    """all-tile indices of the level-0 cells (leaf segment, then inner segment)"""
    segs = []
    for b, c in ((o.leaf_begin[0], o.leaf_count[0]), (o.inner_begin[0], o.inner_count[0])):
        segs.append(np.arange(b * o.B3, (b + c) * o.B3))
    return np.concatenate(segs)


@pytest.mark.parametrize("seed", range(3))
def test_direct_coarsest_is_exact_level0_solve(seed):
    """Dirichlet walls (nonsingular A^0): the direct coarsest solve returns the exact solution of
    A^0 u = b^0 over the active level-0 cells — checked against numpy's dense solve of the level
    operator assembled column by column (random graded trees, non-cubic level 0, random masks
    and face weights)."""
    from tests.helpers import dense_level
    rng = np.random.default_rng(40 + seed)
    ext = [(1, 1, 1), (2, 1, 1), (1, 2, 2)][seed]
    t = random_graded_tree(rng, 1, 2, 0.3, ext=ext)
    o = Oracle(t, ext=ext, B=4)
    kind = rng.choice([0, 1, 2], size=o.N, p=[0.85, 0.05, 0.1]).astype(np.uint8)
    w = (0.1 + 0.9 * rng.random((6, o.N))).astype(np.float32)
    o.setup(kind, w)
    cells = _level0(o)
    cf = o.coefs()
    act = cells[cf[cells, 0] != 0]
    A = dense_level(o, 0, act)
    b = np.zeros(o.T * o.B3)
    b[cells] = rng.standard_normal(len(cells))
    u = o.direct_coarsest(b, np.zeros(o.T * o.B3))
    ref = np.linalg.solve(A, b[act])
    assert np.abs(u[act] - ref).max() <= 1e-10 * np.abs(ref).max()
    inact = cells[cf[cells, 0] == 0]
    assert np.all(u[inact] == 0.0)


def test_direct_coarsest_floating_components_pseudo_inverse():
    """Singular level 0: one level-0 tile (L = 0, B = 8), Dirichlet walls, a Neumann shell
    that seals a 2x2x2 fluid pocket off from the rest (a floating component: A^0 1 = 0 on it,
    P:L343) — the direct solve equals the minimum-norm solution pinv(A^0) b (numpy), i.e. the
    exact inverse on the wall-connected component and the zero-mean solution of the
    mean-free rhs on the pocket."""
    from tests.helpers import dense_level
    rng = np.random.default_rng(3)
    o = Oracle(np.array([[0, 0, 0, 0]], dtype=np.int32))
    X, Y, Z = np.meshgrid(np.arange(8), np.arange(8), np.arange(8), indexing="ij")
    X, Y, Z = (a.transpose(2, 1, 0).ravel() for a in (X, Y, Z))  # natural order x + 8y + 64z
    shell = (np.maximum(np.maximum(np.abs(X - 3.5), np.abs(Y - 3.5)), np.abs(Z - 3.5)) == 1.5)
    kind = np.where(shell, 2, 0).astype(np.uint8)
    o.setup(kind)
    cells = _level0(o)
    act = cells[o.coefs()[cells, 0] != 0]
    A = dense_level(o, 0, act)
    assert np.linalg.matrix_rank(A) == len(act) - 1  # exactly one floating component
    b = np.zeros(o.T * o.B3)
    b[act] = rng.standard_normal(len(act))
    u = o.direct_coarsest(b, np.zeros(o.T * o.B3))
    ref = np.linalg.pinv(A) @ b[act]
    assert np.abs(u[act] - ref).max() <= 1e-10 * np.abs(ref).max()


def test_direct_coarsest_single_level_pcg_one_iteration():
    """A one-level tree (L = 0): the FAS cycle with a direct coarsest solve is A^{-1}, so PCG
    converges in one iteration (Alg. 1), while the smoothing-only cycle needs several."""
    rng = np.random.default_rng(8)
    o = Oracle(np.array([[0, 0, 0, 0]], dtype=np.int32))
    kind = rng.choice([0, 1, 2], size=o.N, p=[0.9, 0.05, 0.05]).astype(np.uint8)
    o.setup(kind)
    b = rng.standard_normal(o.N) * (kind == 0)
    d = o.pcg(b, rtol=1e-10, coarsest="direct")
    s = o.pcg(b, rtol=1e-10)
    assert d["status"] == "OK" and d["iters"] == 1
    assert s["iters"] > 1


@pytest.mark.parametrize("mu", [1, 2])
def test_direct_coarsest_cycle_converges_no_slower(mu):
    """On an adaptive Dirichlet problem the cycle with the exact coarsest solve is at least as
    good a preconditioner as the 10-iteration smoother: PCG iterations no larger, solutions
    equal within the solve tolerance."""
    cfg = make_config("sphere_small_dir")
    o = Oracle(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
    o.setup(cfg["kind"], cfg["w"])
    b = cfg["b"].astype(np.float64)
    d = o.pcg(b, rtol=1e-8, mu=mu, coarsest="direct")
    s = o.pcg(b, rtol=1e-8, mu=mu)
    assert d["iters"] <= s["iters"]
    assert np.linalg.norm(d["x"] - s["x"]) <= 1e-6 * np.linalg.norm(s["x"])
