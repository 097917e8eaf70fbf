"""One apply, one V/W-cycle and one PCG solve of a small config for compute-sanitizer
(racecheck / synccheck / memcheck): the in-place colour passes, the shuffles of the row
kernels, the dense coarse cycle's barriers and the tile-layout sub-cycle.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py tank_small [ENV=VAL ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
for kv in sys.argv[2:]:
    k, v = kv.split("=", 1)
    os.environ[k] = v
import numpy as np
import torch

import paper_2604_18886_b200 as om
from octgen import make_config

name = sys.argv[1] if len(sys.argv) > 1 else "tank_small"
cfg = make_config(name)
tree = om.Tree(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
frac = None if cfg["w"] is None else torch.from_numpy(np.ascontiguousarray(cfg["w"])).cuda()
h = om.Hierarchy(tree, torch.from_numpy(cfg["kind"]).cuda(), face_frac=frac, mu=cfg["mu"])
r = torch.from_numpy(np.random.default_rng(1).standard_normal(tree.N).astype(np.float32)).cuda()
u = torch.zeros_like(r)
h.apply(r, u)
h.vcycle(r, u)
b = torch.from_numpy(cfg["b"]).cuda()
x = torch.zeros_like(b)
rep = h.pcg_solve(b, x, rtol=1e-6, max_iters=3)
torch.cuda.synchronize()
print(name, "iters", rep["iters"], "ok")
