"""GPU parity of the cycle variants through the C ABI against the fp64 oracle:
literal Alg. 3 coefficients (P:L499-517 as printed), the standard mu-cycle Alg. 2 with beta
at prolongation (uniform trees), and multigrid as a standalone solver (P:L145,
P:L411, beta = 1).  Bars as tests/test_gpu_parity.py."""
import numpy as np
import pytest

from octgen import make_config
from oracle.oracle import Oracle
from tests.helpers import random_graded_tree

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


def _pair(om, cfg, oracle_kw=None, **mg):
    tree = om.Tree(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
    kind = torch.from_numpy(cfg["kind"]).to(DEV)
    frac = None if cfg["w"] is None else torch.from_numpy(np.ascontiguousarray(cfg["w"])).to(DEV)
    h = om.Hierarchy(tree, kind, face_frac=frac, **mg)
    o = Oracle(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
    o.setup(cfg["kind"], cfg["w"], **(oracle_kw or {}))
    return tree, h, o


@pytest.mark.parametrize("seed", range(3))
def test_literal_coarsening_matches_oracle(om, seed):
    rng = np.random.default_rng(40 + seed)
    tiles = random_graded_tree(rng, 1, 3, 0.35)
    N = len(tiles) * 512
    kind = rng.choice([0, 1, 2], size=N, p=[0.8, 0.1, 0.1]).astype(np.uint8)
    w = rng.random((6, N)).astype(np.float32)
    tree = om.Tree(tiles)
    h = om.Hierarchy(tree, torch.from_numpy(kind).to(DEV), None, torch.from_numpy(w).to(DEV), coarsen_literal=True)
    o = Oracle(tiles)
    o.setup(kind, w, coarsen_literal=True)
    g, r = h.export_coefs().astype(np.float64), o.coefs()
    scale = np.abs(r).max(axis=1, keepdims=True) + 1e-30
    assert (np.abs(g - r) / scale).max() <= 5e-6
    assert np.array_equal(g[:, 0] != 0, r[:, 0] != 0)
    # the literal reading really differs from the default on these masks (Dirichlet cells)
    o2 = Oracle(tiles)
    o2.setup(kind, w)
    assert not np.array_equal(o2.coefs(), r)


@pytest.mark.parametrize("name", ["uniform32", "uniform64_dir"])
@pytest.mark.parametrize("mu", [1, 2])
def test_alg2_cycle_matches_oracle(om, name, mu):
    cfg = make_config(name)
    tree, h, o = _pair(om, cfg, mu=mu, form="alg2")
    r = np.random.default_rng(7).standard_normal(o.N).astype(np.float32)
    u = torch.zeros(o.N, device=DEV)
    h.vcycle(torch.from_numpy(r).to(DEV), u)
    ref = o.vcycle(r.astype(np.float64), form="alg2", mu=mu)
    assert _rel(u.cpu().numpy().astype(np.float64), ref) <= 1e-5
    # on a uniform tree Alg. 2 and Alg. 4 are the same linear map (oracle pin); the GPU agrees
    ref4 = o.vcycle(r.astype(np.float64), mu=mu)
    assert _rel(u.cpu().numpy().astype(np.float64), ref4) <= 1e-5


def test_alg2_rejects_adaptive_tree(om):
    cfg = make_config("sphere_small")
    with pytest.raises(om.OctmgError):
        _pair(om, cfg, form="alg2")


def test_alg2_pcg_matches_oracle(om):
    cfg = make_config("uniform64_dir")
    tree, h, o = _pair(om, cfg, form="alg2")
    b = torch.from_numpy(cfg["b"]).to(DEV)
    x = torch.zeros_like(b)
    rep = h.pcg_solve(b, x, rtol=1e-6)
    ref = o.pcg(cfg["b"].astype(np.float64), rtol=1e-6, precond="alg2")
    assert rep["converged"] and abs(rep["iters"] - ref["iters"]) <= 1
    assert _rel(x.cpu().numpy().astype(np.float64), ref["x"]) <= 1e-5


@pytest.mark.parametrize("name,mu", [("uniform32", 1), ("sphere_small_dir", 1), ("tank_small", 2)])
def test_standalone_mg_matches_oracle(om, name, mu):
    cfg = make_config(name)
    tree, h, o = _pair(om, cfg, mu=mu, beta=1.0)
    b = torch.from_numpy(cfg["b"]).to(DEV)
    x = torch.zeros_like(b)
    rep = h.mg_solve(b, x, rtol=1e-6, max_iters=400)
    ref = o.mg_solve(cfg["b"].astype(np.float64), rtol=1e-6, mu=mu, beta=1.0, max_iters=400)
    assert rep["converged"] and ref["status"] == "OK"
    assert abs(rep["iters"] - ref["iters"]) <= 1, (rep["iters"], ref["iters"])
    xg, xr = x.cpu().numpy().astype(np.float64), ref["x"]
    if cfg["bc"] == "neumann_layer":  # unique up to a constant
        act = o.coefs()[:o.N, 0] != 0
        xg = xg - xg[act].mean() * act
        xr = xr - xr[act].mean() * act
    assert _rel(xg, xr) <= 1e-5, _rel(xg, xr)
    # the per-iteration residual history follows the oracle's
    n = min(len(rep["history"]), len(ref["history"]))
    assert np.allclose(rep["history"][:n], ref["history"][:n], rtol=1e-3, atol=1e-7)


# ---------------------------------------------------------------------------------------
# direct coarsest solve (Alg. 4 line 4; DESIGN reading 9b)
# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("env", [{}, {"OCTMG_SUBCYCLE": "0"}])
@pytest.mark.parametrize("name,mu", [("cfg1_octant", 1), ("sphere_small_dir", 2), ("tank_small", 2),
                                     ("uniform32", 1), ("sphere_small", 2)])
def test_direct_coarsest_cycle_and_pcg_match_oracle(om, name, mu, env, monkeypatch):
    """The cycle with the direct level-0 solve (on chip in the sub-cycle, or the standalone
    k_coarse_direct launch with OCTMG_SUBCYCLE=0) against the oracle's: Dirichlet problems
    (nonsingular level 0) and pure-Neumann ones (one floating component: the minimum-norm
    solution), mu = 1, 2; the cycle <= 1e-5 and PCG within +-1 iterations, <= 1e-5."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    cfg = make_config(name)
    tree, h, o = _pair(om, cfg, mu=mu, coarsest="direct")
    rng = np.random.default_rng(21)
    act = o.coefs_diag_leaf() != 0
    r = (rng.standard_normal(o.N) * act).astype(np.float32)
    z = torch.zeros(o.N, device=DEV)
    h.vcycle(torch.from_numpy(r).to(DEV), z)
    zr = o.vcycle(r.astype(np.float64), mu=mu, coarsest="direct")
    assert _rel(z.cpu().numpy().astype(np.float64), zr) <= 1e-5
    b = torch.from_numpy(cfg["b"]).to(DEV)
    x = torch.zeros_like(b)
    rep = h.pcg_solve(b, x, rtol=1e-6)
    ref = o.pcg(cfg["b"].astype(np.float64), rtol=1e-6, mu=mu, coarsest="direct")
    assert rep["converged"] and abs(rep["iters"] - ref["iters"]) <= 1
    xg, xr = x.cpu().numpy().astype(np.float64), ref["x"]
    if not any(cfg["wall_bc"]):
        xg, xr = xg - xg[act].mean() * act, xr - xr[act].mean() * act
    assert _rel(xg, xr) <= 1e-5


def test_direct_coarsest_single_level_one_iteration(om):
    """One-level tree: M = A^{-1} (to fp32 rounding), so PCG reaches 1e-6 in one iteration."""
    rng = np.random.default_rng(8)
    tiles = np.array([[0, 0, 0, 0]], dtype=np.int32)
    tree = om.Tree(tiles)
    kind = rng.choice([0, 1, 2], size=512, p=[0.9, 0.05, 0.05]).astype(np.uint8)
    h = om.Hierarchy(tree, torch.from_numpy(kind).to(DEV), coarsest="direct")
    b = torch.from_numpy((rng.standard_normal(512) * (kind == 0)).astype(np.float32)).to(DEV)
    x = torch.zeros_like(b)
    rep = h.pcg_solve(b, x, rtol=1e-5)
    assert rep["converged"] and rep["iters"] == 1


def test_direct_coarsest_rejects_large_level0(om):
    """More than 4096 level-0 cells (ext product > 8): OCTMG_E_INVALID."""
    from octgen import uniform_tiles, canonical_order
    ext = (3, 3, 1)
    tiles = uniform_tiles(0, ext)
    tiles = tiles[canonical_order(tiles)]
    tree = om.Tree(tiles, ext)
    with pytest.raises(Exception):
        om.Hierarchy(tree, torch.zeros(tree.N, dtype=torch.uint8, device=DEV), coarsest="direct")
