"""GPU parity of the projection operators (octmg_divergence / octmg_subtract_gradient,
SURVEY 8(f)-2) against the fp64 oracle, and the projection step of the paper's static tank
test: solve A p = div(u), subtract G p, the divergence left is the residual."""
import numpy as np
import pytest

from octgen import make_config
from oracle.oracle import Oracle
from tests.helpers import random_graded_tree

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
DEV = "cuda:0"
TANK_WALLS = (0, 0, 0, 1, 0, 0)


@pytest.fixture(scope="module")
def om():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2604_18886_b200._build import build_library
    build_library()
    import paper_2604_18886_b200 as m
    return m


def _tank(om, name, radius=0.3):
    cfg = make_config(name, with_fields=False)
    tree = om.Tree(cfg["tiles"], cfg["ext"], TANK_WALLS)
    kind, frac, b = om.tank_fields(tree, (0.5, 0.5, 0.5), radius)
    h = om.Hierarchy(tree, kind, face_frac=frac, mu=2)
    o = Oracle(cfg["tiles"], cfg["ext"], TANK_WALLS)
    o.setup(kind.cpu().numpy(), frac.cpu().numpy())
    return tree, h, o, kind, frac, b


@pytest.mark.parametrize("name", ["tank_small", "tank_mid"])
def test_divergence_and_gradient_match_oracle(om, name):
    tree, h, o, kind, frac, b = _tank(om, name)
    rng = np.random.default_rng(1)
    u = rng.standard_normal((6, o.N)).astype(np.float32)
    p = rng.standard_normal(o.N).astype(np.float32)
    fr = frac.cpu().numpy()
    ug = torch.from_numpy(u).to(DEV)
    d = torch.zeros(o.N, device=DEV)
    h.divergence(ug, d, face_frac=frac)
    dref = o.divergence(fr, u.astype(np.float64))
    assert np.abs(d.cpu().numpy() - dref).max() <= 2e-6 * np.abs(dref).max()
    h.subtract_gradient(torch.from_numpy(p).to(DEV), ug, kind, face_frac=frac)
    uref = o.subtract_gradient(fr, p.astype(np.float64), u.astype(np.float64))
    ug_h = ug.cpu().numpy().astype(np.float64)
    scale = np.abs(uref).max()
    assert np.abs(ug_h - uref).max() <= 1e-5 * scale


def test_gpu_identity_div_of_projection(om):
    """div(u - G p) = div(u) - A p with the device operators (octmg_apply), random data."""
    tree, h, o, kind, frac, b = _tank(om, "tank_mid")
    rng = np.random.default_rng(2)
    u = torch.from_numpy(rng.standard_normal((6, o.N)).astype(np.float32)).to(DEV)
    p = torch.from_numpy(rng.standard_normal(o.N).astype(np.float32)).to(DEV)
    d0, d1, Ap = (torch.zeros(o.N, device=DEV) for _ in range(3))
    h.divergence(u, d0, face_frac=frac)
    h.apply(p, Ap)
    h.subtract_gradient(p, u, kind, face_frac=frac)
    h.divergence(u, d1, face_frac=frac)
    err = (d1 - (d0 - Ap)).abs().max().item()
    assert err <= 1e-5 * (d0.abs().max().item() + Ap.abs().max().item())


def test_tank_projection_step(om):
    """Unit downward velocity, W-cycle PCG to 1e-6 on b = div(u) (= the tank rhs), then
    u -= G p: the divergence left is the solve's residual (1e-6 ||div u||) plus the fp32
    rounding of u' = u + F/S summed over the faces (~1e-7 |u| h^2 per face, ~1e-4 ||div u||
    in the 2-norm here); the oracle's fp64 projection leaves ~the residual; the projected
    field matches the oracle's."""
    tree, h, o, kind, frac, b = _tank(om, "tank_mid")
    N = tree.N
    u = torch.zeros((6, N), device=DEV)
    u[2] = -1.0
    u[3] = -1.0
    d = torch.zeros(N, device=DEV)
    h.divergence(u, d, face_frac=frac)
    act = torch.from_numpy(o.coefs()[:N, 0] != 0).to(DEV)
    assert torch.allclose(d[act], b[act], rtol=1e-5, atol=1e-9)
    p = torch.zeros(N, device=DEV)
    rep = h.pcg_solve(d, p, rtol=1e-6)
    assert rep["converged"]
    h.subtract_gradient(p, u, kind, face_frac=frac)
    d2 = torch.zeros(N, device=DEV)
    h.divergence(u, d2, face_frac=frac)
    assert d2.norm().item() <= 1e-3 * d.norm().item()
    ref = o.pcg(b.cpu().numpy().astype(np.float64), rtol=1e-6, mu=2)
    u0 = np.zeros((6, N))
    u0[2] = u0[3] = -1.0
    uref = o.subtract_gradient(frac.cpu().numpy(), ref["x"], u0)
    assert np.abs(u.cpu().numpy() - uref).max() <= 1e-4
    dref = o.divergence(frac.cpu().numpy(), uref)
    assert np.linalg.norm(dref) <= 2e-6 * np.linalg.norm(b.cpu().numpy())
