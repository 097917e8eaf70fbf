"""Oracle tree pins: brute force on tiny trees, error classes, determinism (SURVEY c-1)."""
import numpy as np
import pytest

from octgen import octant_tiles, sphere_band_tiles, uniform_tiles
from oracle.oracle import Oracle, OracleError
from tests.helpers import brute_force_tables, random_graded_tree


@pytest.mark.parametrize("seed", range(6))
def test_tables_match_brute_force(seed):
    rng = np.random.default_rng(seed)
    tiles = random_graded_tree(rng, l0=1, lmax=3, p_refine=0.35)
    o = Oracle(tiles)
    tb = o.tables()
    order, nbr, parent, child = brute_force_tables(tiles)
    assert np.array_equal(tb["tiles"], order)
    assert np.array_equal(tb["nbr"], nbr)
    assert np.array_equal(tb["parent"], parent)
    assert np.array_equal(tb["child"], child)


def test_segments_and_counts():
    o = Oracle(octant_tiles(1))
    assert (o.L, o.NL, o.NI) == (2, 15, 2)
    assert list(o.leaf_count) == [0, 7, 8]
    assert list(o.inner_count) == [1, 1, 0]
    assert o.leaf_begin[2] == 0 and o.leaf_begin[1] == 8


def test_sphere_band_accepted_and_volume():
    t = sphere_band_tiles(3, 2, r=0.25)
    o = Oracle(t)
    assert o.NL == 3368
    vol = sum(8.0 ** (-int(l)) for l in t[:, 0])
    assert vol == pytest.approx(1.0, abs=0)


def test_error_classes():
    t = uniform_tiles(1)
    with pytest.raises(OracleError) as e:
        Oracle(t[1:])
    assert e.value.status == "GAP"
    with pytest.raises(OracleError) as e:
        Oracle(np.concatenate([t, t[:1]]))
    assert e.value.status == "OVERLAP"
    with pytest.raises(OracleError) as e:
        Oracle(np.concatenate([t, [[0, 0, 0, 0]]]))
    assert e.value.status == "OVERLAP"
    bad = t.copy()
    bad[0, 1] = 5
    with pytest.raises(OracleError) as e:
        Oracle(bad)
    assert e.value.status == "INVALID"
    ung = sphere_band_tiles(3, 2, r=0.25, repair=False)
    with pytest.raises(OracleError) as e:
        Oracle(ung)
    assert e.value.status == "NOT_GRADED"


def test_rebuild_is_bit_identical():
    rng = np.random.default_rng(3)
    tiles = random_graded_tree(rng, 1, 3, 0.4)
    a = Oracle(tiles).tables()
    b = Oracle(tiles[::-1].copy()).tables()
    for k in a:
        assert np.array_equal(a[k], b[k])
