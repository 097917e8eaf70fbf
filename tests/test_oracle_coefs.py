"""Oracle coefficient pins: Eq. 3 closed forms, coarse constants,
Alg. 3 == strict Galerkin triple product R A P over fluid DOFs (Eq. 7-8, P:L401-405,
P:L447-455) for random fluid/Dirichlet/Neumann masks and random face weights."""
import numpy as np
import pytest

from octgen import sphere_band_tiles, uniform_tiles, canonical_order, octant_tiles
from oracle.oracle import Oracle
from tests.helpers import dense_level


def _sorted(t):
    return t[canonical_order(t)]


def test_all_fluid_coefficients_every_level():
    """All-fluid, Dirichlet walls: every leaf and inner cell at level l carries (6h_l, -h_l)
    (P:L323-324 leaf; P:L460 coarse 12h/-2h in fine units = 6h_l/-h_l), zero on wall faces."""
    for tiles in (octant_tiles(1), sphere_band_tiles(2, 2, r=0.25)):
        o = Oracle(_sorted(tiles))
        o.setup()
        cf = o.coefs()
        X, Y, Z, lev = o.cell_coords()
        h = np.ldexp(1.0, -lev) / 8
        assert np.allclose(cf[:, 0], 6 * h, rtol=0, atol=1e-15)
        for a, P in enumerate((X, Y, Z)):
            expect = np.where(P == 0, 0.0, -h)
            assert np.allclose(cf[:, 1 + a], expect, rtol=0, atol=1e-15)


def _one_cell_kind_case(k):
    t = _sorted(uniform_tiles(0))
    kind = np.zeros(512, dtype=np.uint8)
    c0 = 3 + 8 * 3 + 64 * 3
    kind[c0] = k
    o = Oracle(t)
    o.setup(kind)
    return o.coefs(), c0


def test_neumann_and_dirichlet_neighbour_rules():
    h = 1 / 8
    cf, c0 = _one_cell_kind_case(2)  # Neumann cell
    xp = c0 + 1
    assert cf[xp, 0] == pytest.approx(5 * h)       # one Neumann neighbour -> 5h
    assert cf[xp, 1] == 0.0                        # cross term zeroed
    assert np.all(cf[c0] == 0.0)
    cf, c0 = _one_cell_kind_case(1)  # Dirichlet cell
    assert cf[xp, 0] == pytest.approx(6 * h)       # Dirichlet keeps 6h
    assert cf[xp, 1] == pytest.approx(-h)          # and the -h cross term
    assert cf[c0, 0] == 0.0 and cf[c0, 1] == pytest.approx(-h)


def _rap_case(rng, B, level, walls):
    t = _sorted(uniform_tiles(level))
    o = Oracle(t, wall_bc=walls, B=B)
    N = o.N
    kind = rng.choice([0, 1, 2], size=N, p=[0.6, 0.2, 0.2]).astype(np.uint8)
    w = rng.random((6, N)).astype(np.float32)
    w[rng.random((6, N)) < 0.1] = 0.0
    o.setup(kind, w)
    X, Y, Z, lev = o.cell_coords()
    fine = np.where(lev == level)[0]
    coarse = np.where(lev == level - 1)[0]
    cf = o.coefs()
    Af = dense_level(o, level, fine)
    Ac = dense_level(o, level - 1, coarse)
    # P: active fine cell -> its parent (constant prolongation)
    cpos = {(X[j], Y[j], Z[j]): n for n, j in enumerate(coarse)}
    P = np.zeros((len(fine), len(coarse)))
    for n, i in enumerate(fine):
        if cf[i, 0] != 0.0:
            P[n, cpos[(X[i] >> 1, Y[i] >> 1, Z[i] >> 1)]] = 1.0
    RAP = P.T @ Af @ P / 2.0     # R = P^T / alpha, alpha = 2
    scale = np.abs(Af).max()
    return RAP, Ac, scale


@pytest.mark.parametrize("B,level", [(2, 2), (4, 1), (2, 3)])
def test_alg3_equals_galerkin_triple_product(B, level):
    rng = np.random.default_rng(100 * B + level)
    n_masks = {(2, 2): 120, (4, 1): 60, (2, 3): 8}[(B, level)]
    for m in range(n_masks):
        walls = tuple(int(v) for v in rng.integers(0, 2, size=6))
        RAP, Ac, scale = _rap_case(rng, B, level, walls)
        err = np.abs(RAP - Ac).max() / scale
        assert err < 1e-12, (m, err)


def test_uniform_level_operator_symmetric_psd():
    rng = np.random.default_rng(7)
    for walls in ((1,) * 6, (0,) * 6):
        t = _sorted(uniform_tiles(2))
        o = Oracle(t, wall_bc=walls, B=2)
        kind = rng.choice([0, 1, 2], size=o.N, p=[0.7, 0.15, 0.15]).astype(np.uint8)
        w = rng.random((6, o.N)).astype(np.float32)
        o.setup(kind, w)
        cells = np.arange(o.N)
        A = dense_level(o, o.L, cells)
        assert np.abs(A - A.T).max() <= 1e-14 * np.abs(A).max()
        act = o.coefs()[:o.N, 0] != 0
        ev = np.linalg.eigvalsh(A[np.ix_(act, act)])
        assert ev.min() > -1e-12 * ev.max()          # PSD
        if walls[0] == 1:
            assert ev.min() > 1e-10 * ev.max()       # PD with Dirichlet
