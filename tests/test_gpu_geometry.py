"""GPU parity of the cut-cell geometry (octmg_tank_fields) against the fp64
oracle: kinds bit-exact, face fractions and right-hand side within fp32 rounding; at
BASELINE config 5's full size (1.64M leaf tiles) on a random sample of tiles the oracle
computes one by one; and a solve on the device-generated fields matches the oracle's."""
import numpy as np
import pytest

from octgen import make_config
from oracle.oracle import Oracle, tank_fields as oracle_tank_fields

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
DEV = "cuda:0"


@pytest.fixture(scope="module")
def om():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2604_18886_b200._build import build_library
    build_library()
    import paper_2604_18886_b200 as m
    return m


def _check(kg, wg, bg, ko, wo, bo):
    assert np.array_equal(kg, ko)
    assert np.abs(wg - wo).max() <= 1e-6
    assert np.abs(bg - bo).max() <= 1e-9


@pytest.mark.parametrize("name,centre,radius", [("tank_small", (0.5, 0.5, 0.5), 0.3),
                                                ("tank_mid", (0.45, 0.52, 0.5), 0.31),
                                                ("uniform32", (0.5, 0.5, 0.5), 0.0)])
def test_tank_fields_match_oracle(om, name, centre, radius):
    cfg = make_config(name, with_fields=False)
    tree = om.Tree(cfg["tiles"], cfg["ext"], (0, 0, 0, 1, 0, 0))
    kind, frac, b = om.tank_fields(tree, centre, radius)
    torch.cuda.synchronize()
    ko, wo, bo = oracle_tank_fields(cfg["tiles"], centre=centre, radius=radius)
    _check(kind.cpu().numpy(), frac.cpu().numpy(), b.cpu().numpy(), ko, wo, bo)


@pytest.mark.slow
def test_tank_fields_full_size_cfg5_sampled(om):
    """BASELINE config 5 (l0 = 4..9, r = 0.35, 838.8M leaf cells): device fields of all
    1,638,344 leaf tiles; 3000 random tiles recomputed by the oracle (per-tile, independent)."""
    cfg = make_config("cfg5_tank", with_fields=False)
    tiles = cfg["tiles"]
    tree = om.Tree(tiles, cfg["ext"], (0, 0, 0, 1, 0, 0))
    assert tree.N == 838_832_128
    kind, frac, b = om.tank_fields(tree, (0.5, 0.5, 0.5), 0.35)
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    sel = np.sort(rng.choice(len(tiles), 3000, replace=False))
    ko, wo, bo = oracle_tank_fields(tiles[sel], radius=0.35)
    cells = (sel[:, None] * 512 + np.arange(512)[None, :]).ravel()
    idx = torch.from_numpy(cells).to(DEV)
    _check(kind[idx].cpu().numpy(), frac[:, idx].cpu().numpy(), b[idx].cpu().numpy(), ko, wo, bo)
    # every solid cell lies inside the sphere volume: count ~ 4/3 pi r^3 / h^3 per level mix
    assert int((kind == 2).sum()) > 0


def test_solve_on_device_fields_matches_oracle(om):
    cfg = make_config("tank_mid", with_fields=False)
    tree = om.Tree(cfg["tiles"], cfg["ext"], (0, 0, 0, 1, 0, 0))
    kind, frac, b = om.tank_fields(tree, (0.5, 0.5, 0.5), 0.30)
    h = om.Hierarchy(tree, kind, face_frac=frac, mu=2)
    x = torch.zeros_like(b)
    rep = h.pcg_solve(b, x, rtol=1e-6)
    ko, wo, bo = oracle_tank_fields(cfg["tiles"], radius=0.30)
    o = Oracle(cfg["tiles"], cfg["ext"], (0, 0, 0, 1, 0, 0))
    o.setup(ko, wo)
    ref = o.pcg(bo.astype(np.float64), rtol=1e-6, mu=2)
    assert rep["converged"] and abs(rep["iters"] - ref["iters"]) <= 1
    xg = x.cpu().numpy().astype(np.float64)
    assert np.linalg.norm(xg - ref["x"]) / np.linalg.norm(ref["x"]) <= 1e-5


# ---------------------------------------------------------------------------------------
# narrow-band refinement on the device (octmg_band_tiles)
# ---------------------------------------------------------------------------------------
def _sorted_rows(t):
    t = np.asarray(t, dtype=np.int64)
    return t[np.lexsort((t[:, 3], t[:, 2], t[:, 1], t[:, 0]))]


@pytest.mark.parametrize("l0,extra,r,centre,repair", [(2, 2, 0.25, (0.5, 0.5, 0.5), True),
                                                      (3, 2, 0.25, (0.5, 0.5, 0.5), False),
                                                      (2, 3, 0.31, (0.45, 0.52, 0.5), True),
                                                      (4, 3, 0.375, (0.5, 0.5, 0.5), True),   # config 3
                                                      (4, 4, 0.30, (0.5, 0.5, 0.5), True)])   # config 4
def test_band_tiles_match_generator(om, l0, extra, r, centre, repair):
    """The device refinement yields exactly the input generator's tile set (octgen: strict
    box test + grading repair to fixpoint, the same IEEE fp64 operations)."""
    from octgen.trees import sphere_band_tiles, is_graded
    ref = sphere_band_tiles(l0, extra, center=centre, r=r, repair=repair)
    got = om.band_tiles(l0, extra, centre=centre, radius=r, grade_repair=repair)
    assert np.array_equal(_sorted_rows(got), _sorted_rows(ref))
    if repair:
        assert is_graded(got)


def test_band_tiles_table1_counts(om):
    """Table 1's sphere grids (3368 / 15464 / 79080 leaf tiles,
    tests/golden/table1_tiles.json) from the device refinement, and a tree builds on them."""
    import json
    import os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table1_tiles.json")))
    for row in gold["rows"]:
        if "l0" not in row:
            continue
        t = om.band_tiles(row["l0"], 2, radius=gold["sphere_r"])
        assert len(t) == row["tiles"], row
    tree = om.Tree(t, (1, 1, 1), (0, 0, 0, 0, 0, 0))
    assert tree.NL == 79080


@pytest.mark.slow
def test_band_tiles_full_size_cfg5(om):
    """BASELINE config 5's tile list (l0 = 4, 5 extra levels, r = 0.35: 1.64M leaf tiles)
    from the device equals the host generator's."""
    cfg = make_config("cfg5_tank", with_fields=False)
    got = om.band_tiles(4, 5, radius=cfg["radius"])
    assert np.array_equal(_sorted_rows(got), _sorted_rows(cfg["tiles"]))
