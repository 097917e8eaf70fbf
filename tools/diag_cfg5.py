"""Diagnostic: config-5 device solve vs the oracle golden at several rtol; residual histories."""
import os, sys, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from octgen import make_config
from oracle.oracle import tank_fields
from paper_2604_18886_b200 import octmg as om
gold = np.load(os.path.join(ROOT, "tests", "golden", "cfg5_oracle.npz"))
name = sys.argv[1] if len(sys.argv) > 1 else "cfg5_tank"
cfg = make_config(name, with_fields=False)
kind, w, b = tank_fields(cfg["tiles"], radius=cfg["radius"])
tree = om.Tree(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
h = om.Hierarchy(tree, torch.from_numpy(kind).to("cuda"), face_frac=torch.from_numpy(w).to("cuda"), mu=cfg["mu"])
smp = torch.from_numpy(gold["sample"]).to("cuda")
bd = torch.from_numpy(b).to("cuda")
print("oracle history", gold["history"])
for rtol in (1e-6, 1e-7, 1e-8, 1e-9):
    xg = torch.zeros_like(bd)
    rep = h.pcg_solve(bd, xg, rtol=rtol, max_iters=40)
    e = np.linalg.norm(xg[smp].cpu().numpy().astype(np.float64) - gold["x"]) / np.linalg.norm(gold["x"])
    # true residual through the device apply (fp32)
    y = torch.zeros_like(bd)
    h.apply(xg, y)
    act = torch.from_numpy(kind == 0).to("cuda")
    rt = torch.where(act, bd.double() - y.double(), torch.zeros_like(bd, dtype=torch.float64))
    print(f"rtol {rtol:g}: iters {rep['iters']} status {rep['status']} hist {np.array2string(rep['history'], precision=3)} "
          f"true-res(fp32 apply) {float(rt.norm() / bd.double().norm()):.3e} sampled err vs oracle {e:.3e}", flush=True)
