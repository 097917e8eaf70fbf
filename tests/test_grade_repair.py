"""octmg_grade_repair_host (the library's host-side 2:1 grading repair, SURVEY c-1)
— runs without a GPU.  Pinned by the paper's Table 1 tile counts (the strict
sphere-band refinement plus repair reproduces them exactly), by equality with the plain
Python repair of octgen on random trees, and by gradedness, volume, idempotence and
independence of the input order."""
import json
import os

import numpy as np
import pytest

from octgen import sphere_band_tiles, uniform_tiles
from octgen.trees import grade_repair, is_graded

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def om():
    from paper_2604_18886_b200._build import build_library
    build_library()
    import paper_2604_18886_b200 as m
    return m


def _set(t):
    return {tuple(int(v) for v in row) for row in np.asarray(t)}


def test_table1_counts_from_library_repair(om):
    rows = json.load(open(os.path.join(GOLD, "table1_tiles.json")))["rows"]
    for row in rows:
        if "l0" not in row:
            continue
        raw = sphere_band_tiles(row["l0"], 2, r=0.25, repair=False)
        rep = om.grade_repair_host(raw)
        assert len(rep) == row["tiles"], (row["grid"], len(rep))


@pytest.mark.parametrize("seed", range(6))
def test_repair_matches_python_and_is_graded(om, seed):
    rng = np.random.default_rng(seed)
    ext = (1, 2, 1) if seed % 2 else (1, 1, 1)
    tiles = uniform_tiles(1, ext)
    for _ in range(3):  # random refinement without grading: violations appear
        sel = rng.random(len(tiles)) < 0.25
        par = tiles[sel]
        kids = [np.stack([par[:, 0] + 1, 2 * par[:, 1] + (d & 1), 2 * par[:, 2] + ((d >> 1) & 1),
                          2 * par[:, 3] + (d >> 2)], axis=1) for d in range(8)]
        tiles = np.concatenate([tiles[~sel]] + kids)
    rep = om.grade_repair_host(tiles, ext)
    assert _set(rep) == _set(grade_repair(tiles, ext))
    assert is_graded(rep, ext)
    vol = sum(8.0 ** -int(l) for l in rep[:, 0])
    assert vol == pytest.approx(float(np.prod(ext)))
    assert _set(om.grade_repair_host(rep, ext)) == _set(rep)  # idempotent
    perm = rng.permutation(len(tiles))
    assert _set(om.grade_repair_host(tiles[perm], ext)) == _set(rep)  # order-independent
