import sys; sys.path.insert(0, '/root/repo')
import numpy as np, torch
from tests.test_gpu_gmg import _setup, _rel
import paper_2604_18886_b200 as om
for name, mu in [("tank_small", 1), ("sphere_small_dir", 1)]:
    cfg, tree, h, h0, o = _setup(om, name, mu)
    rng = np.random.default_rng(21)
    act = o.coefs_diag_leaf() != 0
    r = np.where(act, rng.standard_normal(o.N), 0.0).astype(np.float32)
    u = torch.zeros(o.N, device="cuda"); u0 = torch.zeros(o.N, device="cuda")
    h.vcycle(torch.from_numpy(r).cuda(), u); h0.vcycle(torch.from_numpy(r).cuda(), u0)
    torch.cuda.synchronize()
    g, g0 = u.cpu().numpy().astype(np.float64), u0.cpu().numpy().astype(np.float64)
    ref = o.vcycle(r.astype(np.float64), mu=mu)
    from oracle.oracle import Oracle
    o2 = Oracle(cfg["tiles"], cfg["ext"], cfg["wall_bc"]); o2.setup(cfg["kind"], cfg["w"])
    ref0 = o2.vcycle(r.astype(np.float64), mu=mu)
    print(name, "gpu gmg vs oracle gmg", _rel(g, ref), "gpu gal vs oracle gal", _rel(g0, ref0), "gpu gmg vs gpu gal", _rel(g, g0), "oracle gmg vs gal", _rel(ref, ref0))
    import os
    for env in ["OCTMG_COARSE_DENSE=0", "OCTMG_SUBCYCLE=0"]:
        k, v = env.split("="); os.environ[k] = v
        kind = torch.from_numpy(cfg["kind"]).cuda(); frac = torch.from_numpy(np.ascontiguousarray(cfg["w"])).cuda() if cfg["w"] is not None else None
        ki, wi = (om.tank_fields_inner(tree, radius=cfg["radius"]) if cfg["bc"] == "tank" else (torch.zeros(o.NI*512, dtype=torch.uint8, device="cuda"), None))
        h2 = om.Hierarchy(tree, kind, face_frac=frac, mu=mu, gmg=(ki, None, wi))
        u2 = torch.zeros(o.N, device="cuda"); h2.vcycle(torch.from_numpy(r).cuda(), u2); torch.cuda.synchronize()
        print("  ", env, _rel(u2.cpu().numpy().astype(np.float64), ref))
        del os.environ[k]
