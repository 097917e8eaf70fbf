"""Profile one kind of preconditioner application (no convergence needed): per-kernel times."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2604_18886_b200 as om
from octgen import make_config

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2_uniform256"
cfg = make_config(name)
tree = om.Tree(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
frac = None if cfg["w"] is None else torch.from_numpy(np.ascontiguousarray(cfg["w"])).cuda()
h = om.Hierarchy(tree, torch.from_numpy(cfg["kind"]).cuda(), face_frac=frac, mu=cfg["mu"])
b = torch.from_numpy(cfg["b"]).cuda()
u = torch.zeros_like(b)
for _ in range(3):
    h.vcycle(b, u)
torch.cuda.synchronize()
h.profile(True)
for _ in range(5):
    h.vcycle(b, u)
p = h.profile_read()
h.profile(False)
tot = 0
for k, v in p.items():
    if v["launches"]:
        tot += v["ms"]
        print("  %-22s %8.3f ms/cycle  n=%4d  %6.0f GB/s" % (k, v["ms"] / 5, v["launches"] // 5,
                                                         v["bytes"] / max(v["ms"], 1e-9) / 1e6))
print("total %.3f ms per cycle (%s)" % (tot / 5, os.environ.get("OCTMG_RB", "fused")))
