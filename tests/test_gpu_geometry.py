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
