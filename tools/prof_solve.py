"""One warm-up solve + N solves of a config (for ncu launch lists / captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2604_18886_b200 as om
from octgen import make_config

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2_uniform256"
nsolve = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = make_config(name)
tree = om.Tree(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
frac = None if cfg["w"] is None else torch.from_numpy(np.ascontiguousarray(cfg["w"])).cuda()
h = om.Hierarchy(tree, torch.from_numpy(cfg["kind"]).cuda(), face_frac=frac, mu=cfg["mu"])
b = torch.from_numpy(cfg["b"]).cuda()
x = torch.zeros_like(b)
for _ in range(1 + nsolve):
    rep = h.pcg_solve(b, x)
torch.cuda.synchronize()
print(name, rep["iters"], rep["kernel_launches"])
