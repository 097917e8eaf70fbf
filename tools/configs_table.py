"""Write profiles/<tag>_configs.md and <tag>_bench_cfg2.json from gpurun_out/bench*.json
(tools/gpu_final.sh outputs):  python tools/configs_table.py r01"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT, PROF = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"


def line(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


files = [("cfg1_octant", "bench_cfg1_octant.json"), ("cfg2_uniform256", "bench.json"),
         ("cfg3_sphere", "bench_cfg3_sphere.json"), ("cfg4_tank", "bench_cfg4_tank.json"),
         ("cfg5_tank", "bench_cfg5_tank.json")]
rows, classes = [], []
for name, f in files:
    d = line(os.path.join(OUT, f))
    if name == "cfg2_uniform256":
        open(os.path.join(PROF, f"{tag}_bench_cfg2.json"), "w").write(json.dumps(d, indent=1) + "\n")
    k = sorted(d["kernels"].items(), key=lambda kv: -kv[1]["ms_per_solve"])
    c = d["config"]
    rows.append(f"| {name} | {c['leaf_cells']} | {c['pcg_iters']} | {d['ms_per_step']:.2f} | {d['value']:.3e} | "
                f"{d['e2e']['value']:.3e} | {k[0][0]} {k[0][1]['ms_per_solve']:.2f} ms |")
    classes.append(f"- {name}: " + ", ".join(f"{n} {v['ms_per_solve']:.3f} (n={v['launches_per_solve']})" for n, v in k))
md = [f"# {tag}: bench lines of the BASELINE configs on one B200 (final round-1 code)", "",
      "`python bench.py` (config 2, 50 steps) and `python bench.py --config C --steps 5 --warmup 3 --no-cpu-baseline`;",
      "configs 4/5 take kind / face fractions / rhs from the device geometry pipeline (`octmg_tank_fields`).", "",
      "| config | leaf cells | PCG iters | ms / solve | cells/s | e2e cells/s | dominant class (profiling pass) |",
      "|---|---|---|---|---|---|---|", *rows, "",
      "Per-class time per solve (ms; CUDA events around every launch, graph replay off):", "", *classes, "",
      "The W-cycle configs 4/5 are dominated by the coarse levels (per-level launches and the on-chip sub-cycle, "
      "latency-bound); config 3's finest levels carry many ghost (T-junction) tiles on the general stencil path.  "
      "Paper context (RTX 4090): >2e8 cells/s analytic, >7e7 cells/s projection."]
open(os.path.join(PROF, f"{tag}_configs.md"), "w").write("\n".join(md) + "\n")
print("\n".join(rows))
