"""Per-phase cost of the one-CTA dense coarse cycle: the level-1 visit time of config 4 with
nu_coarsest = 10 / 2 and nu_pre = nu_post = 2 / 1 (levels 0-1 in k_coarse_dense,
OCTMG_COARSE_CLUSTER=0), from the per-level event profile."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["OCTMG_COARSE_CLUSTER"] = "0"
import torch

import paper_2604_18886_b200 as om
from octgen import make_config

cfg = make_config("cfg4_tank", with_fields=False)
tree = om.Tree(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
kind, frac, b = om.tank_fields(tree, (0.5, 0.5, 0.5), cfg["radius"])
for nc, nu in ((10, 2), (2, 2), (10, 1), (2, 1)):
    h = om.Hierarchy(tree, kind, face_frac=frac, mu=2, nu_coarsest=nc, nu_pre=nu, nu_post=nu)
    x = torch.zeros_like(b)
    h.pcg_solve(b, x)
    h.profile(True)
    rep = h.pcg_solve(b, x)
    lv = h.profile_read_levels(range(tree.L + 1))
    h.profile(False)
    d = lv[1]["coarse_subcycle"]
    print(f"nu_coarsest {nc} nu {nu}: iters {rep['iters']} level-1 visits {d['launches']} "
          f"{1e3 * d['ms'] / d['launches']:.2f} us per visit", flush=True)
    del h
