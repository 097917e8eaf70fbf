"""Oracle multigrid pins: FAS-style cycle (Alg. 4) == standard cycle with beta at
prolongation (Alg. 2) on uniform trees (P:L864-866 linearity argument; exact, not a
tolerance claim), linearity M(a b1 + b2) = a M b1 + M b2, RBGS fixed point at the exact
composite solution, symmetric preconditioner on uniform trees."""
import numpy as np
import pytest

from octgen import canonical_order, octant_tiles, uniform_tiles
from oracle.oracle import Oracle
from tests.helpers import dense_composite, random_graded_tree


def _sorted(t):
    return t[canonical_order(t)]


@pytest.mark.parametrize("mu", [1, 2])
@pytest.mark.parametrize("seed", range(4))
def test_fas_equals_alg2_on_uniform_trees(mu, seed):
    rng = np.random.default_rng(seed)
    B, level = (2, 3) if seed % 2 else (4, 2)
    walls = tuple(int(v) for v in rng.integers(0, 2, size=6))
    o = Oracle(_sorted(uniform_tiles(level)), wall_bc=walls, B=B)
    kind = rng.choice([0, 1, 2], size=o.N, p=[0.8, 0.1, 0.1]).astype(np.uint8)
    w = rng.random((6, o.N)).astype(np.float32)
    o.setup(kind, w)
    r = rng.standard_normal(o.N)
    z4 = o.vcycle(r, form="fas", mu=mu, beta=2.0)
    z2 = o.vcycle(r, form="alg2", mu=mu, beta=2.0)
    assert np.abs(z4 - z2).max() <= 1e-12 * np.abs(z2).max()


def test_cycle_is_linear_on_adaptive_tree():
    rng = np.random.default_rng(5)
    t = random_graded_tree(rng, 1, 3, 0.35)
    o = Oracle(t)
    kind = rng.choice([0, 1, 2], size=o.N, p=[0.85, 0.05, 0.1]).astype(np.uint8)
    o.setup(kind)
    b1, b2 = rng.standard_normal(o.N), rng.standard_normal(o.N)
    for mu in (1, 2):
        lhs = o.vcycle(2.5 * b1 + b2, mu=mu)
        rhs = 2.5 * o.vcycle(b1, mu=mu) + o.vcycle(b2, mu=mu)
        assert np.abs(lhs - rhs).max() <= 1e-12 * np.abs(rhs).max()
        assert np.all(o.vcycle(np.zeros(o.N), mu=mu) == 0.0)


def test_rbgs_fixed_point_at_exact_composite_solution():
    """u = A^{-1} b (dense) on an adaptive tree; an RBGS colour pass at the finest level,
    with coarse leaves holding the same solution, leaves u unchanged (consistent smoother)."""
    rng = np.random.default_rng(9)
    o = Oracle(_sorted(octant_tiles(1)), B=4)
    o.setup()
    A = dense_composite(o)
    b = rng.standard_normal(o.N)
    x = np.linalg.solve(A, b)
    u_all = np.zeros(o.T * o.B3)
    b_all = np.zeros(o.T * o.B3)
    u_all[:o.N] = x
    b_all[:o.N] = b
    for colour in (0, 1):
        u2 = o.rbgs_pass(o.L, colour, u_all, b_all)
        assert np.abs(u2 - u_all).max() <= 1e-12 * np.abs(x).max()


def test_rbgs_pass_updates_one_colour_by_its_row():
    """A pass touches only cells of its colour at its level, and each updated cell
    satisfies its own row with the other colour fixed (uniform tree: no ghosts)."""
    rng = np.random.default_rng(4)
    o = Oracle(_sorted(uniform_tiles(1)), B=4)
    o.setup()
    X, Y, Z, lev = o.cell_coords()
    u = rng.standard_normal(o.T * o.B3) * (lev == o.L)
    b = rng.standard_normal(o.T * o.B3) * (lev == o.L)
    u2 = o.rbgs_pass(o.L, 0, u, b)
    red = ((X + Y + Z) % 2 == 0) & (lev == o.L)
    assert np.all(u2[~red] == u[~red])
    r = b - o.apply_level(o.L, u2)
    assert np.abs(r[red]).max() <= 1e-13 * np.abs(b).max()


def test_preconditioner_symmetric_on_uniform_tree():
    rng = np.random.default_rng(2)
    o = Oracle(_sorted(uniform_tiles(2)), B=4)
    o.setup()
    for mu in (1, 2):
        b1, b2 = rng.standard_normal(o.N), rng.standard_normal(o.N)
        a = o.vcycle(b1, mu=mu) @ b2
        c = b1 @ o.vcycle(b2, mu=mu)
        assert abs(a - c) <= 1e-10 * abs(a)


@pytest.mark.parametrize("mu", [1, 2])
@pytest.mark.parametrize("seed", range(3))
def test_eq14_children_mean_equals_coarse_value_after_prolongation(mu, seed):
    """Eq. 14: with the FAS update p_i = u_i + (p_P - u*_P) and u*_P the mean
    of the active children, the mean of the active children after every prolongation equals
    the coarse value p_P — on adaptive trees (coarse leaves, T-junctions) with random
    fluid / Dirichlet / Neumann masks, for mu = 1 and 2.  A beta != 1 at prolongation, a
    correction added to inactive children or an Avg over all 8 children would break it."""
    rng = np.random.default_rng(100 + seed)
    t = random_graded_tree(rng, 1, 3, 0.4)
    walls = tuple(int(v) for v in rng.integers(0, 2, size=6))
    o = Oracle(t, wall_bc=walls)
    kind = rng.choice([0, 1, 2], size=o.N, p=[0.8, 0.05, 0.15]).astype(np.uint8)
    w = (0.2 + 0.8 * rng.random((6, o.N))).astype(np.float32)
    o.setup(kind, w)
    o.eq14_check(True)
    o.vcycle(rng.standard_normal(o.N), mu=mu)
    dev, scale = o.eq14_result()
    o.eq14_check(False)
    assert scale > 0.0
    assert dev <= 1e-12 * scale, (dev, scale)


@pytest.mark.parametrize("neumann_side", [False, True])
def test_rbgs_two_cell_system_hand_iterated(neumann_side):
    """Gauss-Seidel by hand on a 2-cell system (SURVEY 8(c-9) 'hand-iterated GS'): one level-0
    tile of 2^3 cells (B = 2, h = 1/2), Dirichlet walls, two x-adjacent fluid cells (red
    (0,0,0), black (1,0,0)), every other cell Dirichlet — or Neumann above the red cell.
    By P:L323-330 the system is [[c0, -h], [-h, 6h]] with c0 = 6h (5h with the Neumann
    neighbour); red pass u0 = (b0 + h u1)/c0, black pass u1 = (b1 + h u0)/(6h)."""
    from fractions import Fraction as F
    o = Oracle(np.array([[0, 0, 0, 0]], dtype=np.int32), B=2)
    kind = np.ones(8, dtype=np.uint8)
    kind[0] = kind[1] = 0          # natural order x + 2y + 4z
    if neumann_side:
        kind[2] = 2                # (0,1,0): Neumann above the red cell
    o.setup(kind)
    h = F(1, 2)
    c0 = 5 * h if neumann_side else 6 * h
    cf = o.coefs()
    assert cf[0, 0] == float(c0) and cf[1, 0] == float(6 * h) and cf[1, 1] == float(-h)
    b0, b1 = F(1), F(-2)
    u0, u1 = F(0), F(0)
    u = np.zeros(8)
    b = np.zeros(8)
    b[0], b[1] = float(b0), float(b1)
    for it in range(4):
        u0 = (b0 + h * u1) / c0
        u = o.rbgs_pass(0, 0, u, b)
        assert abs(u[0] - float(u0)) <= 1e-15 and abs(u[1] - float(u1)) <= 1e-15
        u1 = (b1 + h * u0) / (6 * h)
        u = o.rbgs_pass(0, 1, u, b)
        assert abs(u[1] - float(u1)) <= 1e-15 and abs(u[0] - float(u0)) <= 1e-15
        assert np.all(u[2:] == 0.0)
    # converges to the 2x2 solution
    det = c0 * 6 * h - h * h
    x0, x1 = (b0 * 6 * h + h * b1) / det, (c0 * b1 + h * b0) / det
    for _ in range(40):
        u = o.rbgs_pass(0, 1, o.rbgs_pass(0, 0, u, b), b)
    assert abs(u[0] - float(x0)) <= 1e-13 and abs(u[1] - float(x1)) <= 1e-13
