"""One warm-up solve + N solves of a config with the tank fields generated on the device (for ncu
launch lists / captures of the big W-cycle configs).   python tools/prof_solve_dev.py cfg5_tank 0"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2604_18886_b200 as om
from octgen import make_config

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4_tank"
nsolve = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = make_config(name, with_fields=False)
tree = om.Tree(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
if cfg["bc"] == "tank":
    kind, frac, b = om.tank_fields(tree, (0.5, 0.5, 0.5), cfg["radius"])
else:
    cfg = make_config(name)
    kind = torch.from_numpy(cfg["kind"]).cuda()
    frac = None if cfg["w"] is None else torch.from_numpy(np.ascontiguousarray(cfg["w"])).cuda()
    b = torch.from_numpy(cfg["b"]).cuda()
h = om.Hierarchy(tree, kind, face_frac=frac, mu=cfg["mu"])
x = torch.zeros_like(b)
for _ in range(1 + nsolve):
    rep = h.pcg_solve(b, x)
torch.cuda.synchronize()
print(name, rep["iters"], rep["kernel_launches"])
