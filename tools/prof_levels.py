"""Per-level, per-kernel-class device time of one PCG solve of a BASELINE config (CUDA
events around every launch, graph replay off), plus the timed solve without profiling.

    python tools/prof_levels.py cfg4_tank [out.json]
"""
import json
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
tank = cfg["bc"] == "tank"
if not tank:
    cfg = make_config(name)
tree = om.Tree(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
if tank:
    kind, frac, b = om.tank_fields(tree, (0.5, 0.5, 0.5), cfg["radius"])
else:
    kind = torch.from_numpy(cfg["kind"]).cuda()
    frac = None if cfg["w"] is None else torch.from_numpy(np.ascontiguousarray(cfg["w"])).cuda()
    b = torch.from_numpy(cfg["b"]).cuda()
h = om.Hierarchy(tree, kind, face_frac=frac, mu=cfg["mu"])
x = torch.zeros_like(b)
for _ in range(2):
    rep = h.pcg_solve(b, x)
torch.cuda.synchronize()
t0 = time.perf_counter()
n = 3
for _ in range(n):
    rep = h.pcg_solve(b, x)
torch.cuda.synchronize()
ms = (time.perf_counter() - t0) * 1e3 / n
h.profile(True)
rep = h.pcg_solve(b, x)
tot = h.profile_read()
lv = h.profile_read_levels(range(tree.L + 1) if hasattr(tree, "L") else range(16))
h.profile(False)
print(f"{name}: {tree.N} leaves, {rep['iters']} iterations, {ms:.2f} ms per solve (wall, graph replay)")
out = {"config": name, "ms_per_solve": ms, "iters": rep["iters"], "total": tot, "levels": {}}
for l, d in lv.items():
    if not d:
        continue
    s = sum(v["ms"] for v in d.values())
    out["levels"][l] = d
    parts = ", ".join(f"{k} {v['ms']:.2f} ms/{v['launches']}" for k, v in sorted(d.items(), key=lambda kv: -kv[1]["ms"]))
    print(f"  level {l}: {s:8.2f} ms  ({parts})")
pcg = {k: v["ms"] for k, v in tot.items() if v["launches"] and k in ("apply", "pcg_update", "dot_rz", "project", "init", "p_update")}
print("  pcg vectors:", {k: round(v, 2) for k, v in pcg.items()})
if len(sys.argv) > 2:
    json.dump(out, open(sys.argv[2], "w"), indent=1)
