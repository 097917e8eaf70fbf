"""Bit-identity of two apply variants (env-selected at hierarchy setup) on several configs:
  python tools/apply_ab_check.py OCTMG_APPLY_V=4"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2604_18886_b200 as om
from octgen import make_config

k, v = sys.argv[1].split("=")
dev = torch.device("cuda", 0)
bad = 0
for name in ["uniform64_dir", "sphere_small", "sphere_small_dir", "tank_small", "tank_mid", "cfg1_octant"]:
    cfg = make_config(name)
    tree = om.Tree(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
    kind = torch.from_numpy(cfg["kind"]).to(dev)
    frac = None if cfg["w"] is None else torch.from_numpy(np.ascontiguousarray(cfg["w"])).to(dev)
    g = torch.Generator().manual_seed(1)
    x = (torch.rand(cfg["n_cells"], generator=g) * 2 - 1).to(dev)
    outs, reps = [], []
    for env in ({}, {k: v}):
        old = os.environ.get(k)
        os.environ.pop(k, None)
        os.environ.update(env)
        h = om.Hierarchy(tree, kind, face_frac=frac, mu=cfg["mu"])
        y = torch.empty_like(x)
        h.apply(x, y)
        b = torch.from_numpy(cfg["b"]).to(dev)
        xs = torch.zeros_like(b)
        rep = h.pcg_solve(b, xs)
        torch.cuda.synchronize()
        outs.append(y.cpu())
        reps.append((rep["iters"], rep["rel_residual"], xs.cpu()))
        del h
        os.environ.pop(k, None)
        if old is not None:
            os.environ[k] = old
    same = torch.equal(outs[0], outs[1])
    dx = (reps[0][2] - reps[1][2]).abs().max().item()
    print(f"{name}: apply bit-identical={same}  iters {reps[0][0]} vs {reps[1][0]}  max|dx|={dx:.3e}")
    bad += not same
sys.exit(1 if bad else 0)
