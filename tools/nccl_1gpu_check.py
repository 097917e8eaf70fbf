"""Try the NCCL transport with 2 ranks on ONE GPU (torchrun --nproc-per-node 2, both ranks on
cuda:0) and compare the partitioned solve with the single-process loopback partition.
NCCL may refuse duplicate GPUs; then this only reports that.

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/nccl_1gpu_check.py [config]
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_18886_b200 as om  # noqa: E402
from octgen import make_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "sphere_small"
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
cfg = make_config(name)
dev = torch.device("cuda", 0)
kind = torch.from_numpy(cfg["kind"]).to(dev)
frac = None if cfg["w"] is None else torch.from_numpy(np.ascontiguousarray(cfg["w"])).to(dev)
b = torch.from_numpy(cfg["b"]).to(dev)
try:
    comm = om.NcclComm(rank, world)
except Exception as e:
    print(f"rank {rank}: NCCL comm init failed: {e}", flush=True)
    sys.exit(0)
tree = om.Tree(cfg["tiles"], cfg["ext"], cfg["wall_bc"], comm=comm)
h = om.Hierarchy(tree, kind, face_frac=frac, mu=cfg["mu"])
x = torch.zeros_like(b)
rep = h.pcg_solve(b, x, rtol=1e-6)
lg, rk, nr, ob, oc = h.partition(0)
own = torch.zeros(tree.N, dtype=torch.bool, device=dev)
for bg, ct in zip(ob, oc):
    own[int(bg) * 512:(int(bg) + int(ct)) * 512] = True
# reference: loopback partition with the same part count in this process
tree1 = om.Tree(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
h1 = om.Hierarchy(tree1, kind, face_frac=frac, mu=cfg["mu"], loopback_parts=world)
x1 = torch.zeros_like(b)
rep1 = h1.pcg_solve(b, x1, rtol=1e-6)
xs, x1s = x[own], x1[own]
same = bool(torch.equal(xs, x1s))
print(f"rank {rank}: iters nccl {rep['iters']} loopback {rep1['iters']} rel {rep['rel_residual']:.3e}/"
      f"{rep1['rel_residual']:.3e} owned-cells bit-identical {same} "
      f"maxdiff {float((xs - x1s).abs().max()):.3e}", flush=True)
dist.barrier()
del h, tree
comm = None
dist.destroy_process_group()
