"""GPU parity of the GMG comparison mode (octmg_setup_hierarchy_gmg)
against the oracle's (oracle setup_gmg): the inner cells' tank geometry, the cycle's
grid-assembled coarse records, the cycle and the GMG-preconditioned PCG; the composite operator
is the one octmg_setup_hierarchy assembles; on the cut-cell tank the GMG PCG needs more
iterations than the algebraically consistent cycle on the device too (Fig. 12)."""
import numpy as np
import pytest

from octgen import make_config
from oracle.oracle import Oracle, tank_fields

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


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _setup(om, name, mu=None):
    cfg = make_config(name)
    mu = cfg["mu"] if mu is None else mu
    tree = om.Tree(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
    kind = torch.from_numpy(cfg["kind"]).to(DEV)
    frac = None if cfg["w"] is None else torch.from_numpy(np.ascontiguousarray(cfg["w"])).to(DEV)
    o = Oracle(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
    o.setup(cfg["kind"], cfg["w"])
    inner_tiles = o.tables()["tiles"][o.NL:]
    if cfg["bc"] == "tank":
        ki, wi = om.tank_fields_inner(tree, radius=cfg["radius"])
        ko, wo, _ = tank_fields(inner_tiles, cfg["ext"], radius=cfg["radius"])
        assert np.array_equal(ki.cpu().numpy(), ko)  # bit-exact kinds (fp64 SDF, no FMA)
        assert np.array_equal(wi.cpu().numpy(), wo)
        o.setup_gmg(ko, wo)
    else:  # all-fluid inner cells, w = 1
        ki, wi = torch.zeros(o.NI * 512, dtype=torch.uint8, device=DEV), None
        o.setup_gmg()
    h = om.Hierarchy(tree, kind, face_frac=frac, mu=mu, gmg=(ki, None, wi))
    h0 = om.Hierarchy(tree, kind, face_frac=frac, mu=mu)
    return cfg, tree, h, h0, o


@pytest.mark.parametrize("name", ["tank_small", "sphere_small_dir", "tank_mid"])
def test_gmg_cycle_coefficients_match_oracle(om, name):
    cfg, tree, h, h0, o = _setup(om, name)
    assert np.array_equal(h.export_coefs(), h0.export_coefs())  # the composite operator's store
    g = h.export_cycle_coefs().astype(np.float64)
    r = o.coefs_cycle()
    assert np.array_equal(g[:, 0] != 0, r[:, 0] != 0)
    scale = np.abs(r).max(axis=1, keepdims=True) + 1e-300
    assert (np.abs(g - r) / scale).max() <= 2e-6
    if cfg["bc"] != "tank":  # fluid only: the grid records are the Alg. 3 ones
        assert np.abs(g - h0.export_cycle_coefs()).max() <= 2e-6 * np.abs(r).max()


@pytest.mark.parametrize("name,mu", [("tank_small", 1), ("tank_small", 2), ("sphere_small_dir", 1), ("tank_mid", 2)])
def test_gmg_vcycle_matches_oracle(om, name, mu):
    cfg, tree, h, h0, o = _setup(om, name, mu)
    rng = np.random.default_rng(21)
    act = o.coefs_diag_leaf() != 0
    r = np.where(act, rng.standard_normal(o.N), 0.0).astype(np.float32)
    u = torch.zeros(o.N, device=DEV)
    h.vcycle(torch.from_numpy(r).to(DEV), u)
    torch.cuda.synchronize()
    assert _rel(u.cpu().numpy().astype(np.float64), o.vcycle(r.astype(np.float64), mu=mu)) <= 1e-5


@pytest.mark.parametrize("name", ["tank_small", "tank_mid"])
def test_gmg_pcg_matches_oracle_and_is_slower_on_cut_cells(om, name):
    cfg, tree, h, h0, o = _setup(om, name)
    b = torch.from_numpy(cfg["b"]).to(DEV)
    x = torch.zeros_like(b)
    rep = h.pcg_solve(b, x, rtol=1e-6)
    ref = o.pcg(cfg["b"].astype(np.float64), rtol=1e-6, mu=cfg["mu"], max_iters=200)
    assert rep["converged"] and abs(rep["iters"] - ref["iters"]) <= 1, (rep["iters"], ref["iters"])
    assert _rel(x.cpu().numpy().astype(np.float64), ref["x"]) <= 1e-5
    x0 = torch.zeros_like(b)
    rep0 = h0.pcg_solve(b, x0, rtol=1e-6)
    assert rep["iters"] >= rep0["iters"] + 4, (rep0["iters"], rep["iters"])  # Fig. 12
