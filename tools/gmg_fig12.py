"""Fig. 12 on the device at full size: PCG residual histories of config 4 (cut-cell
tank, 155.2M leaves) with the algebraically consistent cycle (mu = 1, 2) and with the GMG
comparison mode's grid-assembled coarse operators (mu = 1, 2), same composite operator."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2604_18886_b200 as om
from octgen import make_config

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4_tank"
cfg = make_config(name, with_fields=False)
tree = om.Tree(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
kind, frac, b = om.tank_fields(tree, (0.5, 0.5, 0.5), cfg["radius"])
ki, fi = om.tank_fields_inner(tree, (0.5, 0.5, 0.5), cfg["radius"])
print(f"{name}: {tree.N} leaves")
for mode in ("ours", "gmg"):
    for mu in (1, 2):
        gmg = (ki, None, fi) if mode == "gmg" else None
        h = om.Hierarchy(tree, kind, face_frac=frac, mu=mu, gmg=gmg)
        x = torch.zeros_like(b)
        h.pcg_solve(b, x, rtol=1e-6, max_iters=100)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = h.pcg_solve(b, x, rtol=1e-6, max_iters=100)
        torch.cuda.synchronize()
        ms = 1e3 * (time.perf_counter() - t0)
        hist = " ".join(f"{v:.2e}" for v in rep["history"][:12])
        print(f"  {mode:4s} mu={mu}: {rep['iters']:3d} iterations, converged {rep['converged']}, {ms:8.1f} ms  history {hist}",
              flush=True)
        del h
