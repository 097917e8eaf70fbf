"""Writes tests/golden/cfg5_oracle.npz: the fp64 ORACLE's full solve of BASELINE config 5
(cut-cell tank, sphere obstacle r = 0.35, leaf levels 4..9, 838.8M leaf cells, W-cycle
mu = 2, rtol 1e-6) sampled at seeded cells, plus the oracle's composite apply of a seeded
random vector at the same cells.  Calls only oracle/ and octgen/ (the input recipe): no
value here comes from the CUDA path.  Needs ~150 GB of host RAM (run it on the GPU box,
which has 196 GB; ~30 min on 16 cores):

    OMP_NUM_THREADS=16 python tools/oracle_golden_cfg5.py [out.npz]

tests/test_gpu_parity.py::test_full_size_cfg5_parity_vs_oracle_golden compares the device
solve (same oracle-generated fields, checked by their SHA-256) against these samples."""
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from octgen import make_config  # noqa: E402
from oracle.oracle import Oracle, tank_fields  # noqa: E402

N_SAMPLES = 200_000
X_SEED = 11          # random vector of the apply check: default_rng(X_SEED).standard_normal(N, float32)
SAMPLE_SEED = 5


def fields_digest(kind, w, b):
    h = hashlib.sha256()
    for a in (kind, w, b):
        h.update(np.ascontiguousarray(a).view(np.uint8))
    return h.hexdigest()


def main(out, name="cfg5_tank"):
    t0 = time.time()
    cfg = make_config(name, with_fields=False)
    tiles = cfg["tiles"]
    kind, w, b = tank_fields(tiles, radius=cfg["radius"])
    digest = fields_digest(kind, w, b)
    N = len(tiles) * 512
    print(f"fields {time.time() - t0:.0f} s, N = {N}, sha256 {digest}", flush=True)
    o = Oracle(tiles, cfg["ext"], cfg["wall_bc"])
    o.setup(kind, w)
    del w
    act = o.coefs_diag_leaf() != 0.0
    print(f"setup {time.time() - t0:.0f} s, active {int(act.sum())}", flush=True)
    rng = np.random.default_rng(SAMPLE_SEED)
    sample = np.sort(rng.choice(np.flatnonzero(act), N_SAMPLES, replace=False)).astype(np.int64)
    x = np.random.default_rng(X_SEED).standard_normal(N, dtype=np.float32)
    y = o.apply(x.astype(np.float64))
    y_s = y[sample].copy()
    y_norm = float(np.linalg.norm(y))
    del x, y
    print(f"apply {time.time() - t0:.0f} s", flush=True)
    ref = o.pcg(b.astype(np.float64), rtol=1e-6, mu=cfg["mu"])
    xs = ref["x"]
    print(f"pcg {time.time() - t0:.0f} s: {ref['iters']} iterations, rel residual {ref['rel_residual']:.3e}, "
          f"status {ref['status']}", flush=True)
    np.savez_compressed(out, sample=sample, x=xs[sample], x_norm=float(np.linalg.norm(xs[act])),
                        y=y_s, y_norm=y_norm, iters=ref["iters"], rel_residual=ref["rel_residual"],
                        history=ref["history"], n_cells=N, n_active=int(act.sum()), fields_sha256=digest,
                        x_seed=X_SEED, sample_seed=SAMPLE_SEED,
                        config=name, recipe=f"{name}: octgen tiles + oracle tank_fields; Oracle.pcg(rtol=1e-6, mu={cfg['mu']})",
                        seconds=time.time() - t0)
    print("wrote", out, flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "tests", "golden", "cfg5_oracle.npz"),
         *(sys.argv[2:3]))
