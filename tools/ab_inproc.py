"""A/B of env-selected schedule variants in ONE process (the workload is generated once):
  python tools/ab_inproc.py CONFIG 'ENV=V,ENV2=V2' 'ENV=V' ...   ('' = defaults)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2604_18886_b200 as om
from octgen import make_config

name = sys.argv[1]
variants = sys.argv[2:] or [""]
cfg = make_config(name)
dev = torch.device("cuda", 0)
tree = om.Tree(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
kind = torch.from_numpy(cfg["kind"]).to(dev)
frac = None if cfg["w"] is None else torch.from_numpy(np.ascontiguousarray(cfg["w"])).to(dev)
b = torch.from_numpy(cfg["b"]).to(dev)
base_env = dict(os.environ)
ref = None
for v in variants:
    os.environ.clear()
    os.environ.update(base_env)
    for kv in filter(None, v.split(",")):
        k, val = kv.split("=")
        os.environ[k] = val
    h = om.Hierarchy(tree, kind, face_frac=frac, mu=cfg["mu"])
    x = torch.zeros_like(b)
    for _ in range(2):
        rep = h.pcg_solve(b, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 5
    e0.record()
    for _ in range(n):
        rep = h.pcg_solve(b, x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    if ref is None:
        ref = x.clone()
    d = float((x - ref).abs().max())
    h.profile(True)
    h.pcg_solve(b, x)
    prof = h.profile_read()
    h.profile(False)
    print(f"== [{v or 'default'}] {name}: {ms:.3f} ms/solve  {tree.N / ms / 1e6:.3f} Gcells/s  iters {rep['iters']}  "
          f"maxdiff vs first {d:.2e}", flush=True)
    for k, p in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
        if p["launches"]:
            print(f"    {k:22s} {p['ms']:8.3f} ms  n={p['launches']:5d}", flush=True)
    del h
