"""Pins of the workload generators against numbers the paper prints."""
import json
import os

import numpy as np
import pytest

from octgen import (canonical_order, face_fraction_marching_squares, is_graded, make_config,
                    morton3, octant_tiles, random_rhs, sphere_band_tiles, tile_counts_by_level,
                    uniform_tiles)
from octgen.fields import tank_fields, splitmix64_uniform

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_table1_sphere_tile_counts():
    """PAPER.md Table 1 (L1792, L1795, L1798): sphere (3-5)/(4-6)/(5-7) leaf-cell counts."""
    rows = json.load(open(os.path.join(GOLD, "table1_tiles.json")))["rows"]
    for r in rows:
        if "l0" in r:
            t = sphere_band_tiles(r["l0"], 2, r=0.25)
            assert len(t) == r["tiles"], r
            assert len(t) * 512 / 2 ** 20 == pytest.approx(r["cells_M"], abs=5e-6)
            assert is_graded(t)
        else:
            t = uniform_tiles(r["level"])
            assert len(t) * 512 / 2 ** 20 == r["cells_M"]


def test_unrepaired_band_is_not_graded():
    t = sphere_band_tiles(3, 2, r=0.25, repair=False)
    assert len(t) == 2808
    assert not is_graded(t)


def test_config_shapes():
    c1 = make_config("cfg1_octant", with_fields=False)
    assert c1["n_cells"] == 7680 and tile_counts_by_level(c1["tiles"]) == {1: 7, 2: 8}
    c3 = make_config("cfg3_sphere", with_fields=False)
    assert tile_counts_by_level(c3["tiles"]) == {4: 2864, 5: 5616, 6: 23208, 7: 85696}
    assert c3["n_cells"] == 117384 * 512


def test_canonical_order_and_morton():
    t = octant_tiles(1)
    o = t[canonical_order(t)]
    assert list(o[:8, 0]) == [2] * 8 and list(o[8:, 0]) == [1] * 7
    m = morton3(o[:8, 1], o[:8, 2], o[:8, 3])
    assert np.all(np.diff(m.astype(np.int64)) > 0)
    assert morton3(1, 0, 0) == 1 and morton3(0, 1, 0) == 2 and morton3(0, 0, 1) == 4
    assert morton3(2, 0, 0) == 8


def test_marching_squares_fractions():
    phi = np.array([[1, 1, -1, -1], [1, 1, 1, 1], [-1, -1, -1, -1], [1, -1, -1, -1.0]])
    f = face_fraction_marching_squares(phi)
    assert f == pytest.approx([0.5, 1.0, 0.0, 0.125])


def test_splitmix_is_counter_based():
    a = splitmix64_uniform(7, np.arange(10, dtype=np.uint64))
    b = splitmix64_uniform(7, np.arange(5, 10, dtype=np.uint64))
    assert np.array_equal(a[5:], b)
    assert np.all((a > -1) & (a < 1))
    assert not np.array_equal(random_rhs(100, 0), random_rhs(100, 1))


def test_tank_without_obstacle_fields():
    t = uniform_tiles(1)
    t = t[canonical_order(t)]
    kind, w, b = tank_fields(t, radius=0.0)
    assert np.all(kind == 0)
    # bottom cells have w_{y-} = 0 (solid wall), top cells w_{y+} = 1 (open)
    h = 1.0 / 16
    assert np.isclose(b.max(), h * h) and np.isclose(b.min(), 0.0)
