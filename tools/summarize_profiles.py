"""Summarise gpurun_out/ ncu outputs into profiles/ (committed evidence).

  python tools/summarize_profiles.py r01
writes profiles/<tag>_launches.csv (trimmed launch list of the bench command),
profiles/<tag>_launch_shares.md, profiles/<tag>_ncu_full.md and updates
profiles/roofline_traffic.json (ncu DRAM bytes per launch of the dominant kernel).
"""
import collections
import csv
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"


def short(name):
    n = name.split("(")[0].replace("void ", "").strip()
    for p in ("octmg::", "(anonymous namespace)::", "<unnamed>::"):
        n = n.replace(p, "")
    return n


def launches():
    path = os.path.join(OUT, "launches_bench.csv")
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, gi, vi, mi = (hdr.index(k) for k in ("Kernel Name", "Grid Size", "Metric Value", "Metric Name"))
    recs = [(short(r[ki]), r[gi], float(r[vi].replace(",", ""))) for r in rows[hi + 1:] if r[mi] == "gpu__time_duration.sum"]
    with open(os.path.join(PROF, f"{tag}_launches.csv"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none "
                "OCTMG_GRAPH_LOOP=0 python bench.py --steps 3 --warmup 3 --no-cpu-baseline (cold-cache, serialised; "
                "host-driven PCG loop so ncu lists the loop body)\n")
        f.write("idx,kernel,grid,ns\n")
        for i, (k, g, t) in enumerate(recs):
            f.write(f"{i},{k},\"{g}\",{t:.0f}\n")
    # the timed region: the 3 solves after the 3 warm-up solves (k_init marks each solve)
    inits = [i for i, r in enumerate(recs) if r[0] == "k_init"]
    start = inits[3] if len(inits) > 6 else inits[0]
    end = inits[6] if len(inits) > 6 else len(recs)
    seg = recs[start:end]
    tot = sum(t for _, _, t in seg)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, g, t in seg:
        key = k + ("  grid=" + g.strip() if k.startswith(("k_pass", "k_restrict", "k_prolong", "k_fasrhs")) else "")
        agg[key][0] += 1
        agg[key][1] += t
    lines = [f"# {tag}: launch shares of the bench's timed solves (ncu launch list, cold-cache, serialised)",
             "", f"solves: {len(inits[3:6]) if len(inits) > 6 else 1}; launches in segment: {len(seg)}; "
             f"sum of kernel time: {tot / 1e6:.3f} ms", "",
             "| kernel | launches | time (ms) | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {k} | {n} | {t / 1e6:.3f} | {100 * t / tot:.1f}% |")
    open(os.path.join(PROF, f"{tag}_launch_shares.md"), "w").write("\n".join(lines) + "\n")


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "sm__inst_executed.sum.pct_of_peak_sustained_elapsed"]


def full():
    out = [f"# {tag}: ncu --set full --clock-control none (one launch each, config 2, level 5 / leaves)", ""]
    traffic = {}
    for rep in sorted(glob.glob(os.path.join(OUT, "full_*.ncu-rep"))):
        k = os.path.basename(rep)[5:-8]
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(txt.splitlines()))
        if len(rows) < 3:
            continue
        hdr, units, r = rows[0], rows[1], rows[2]
        out.append(f"## {k}")
        out.append("")
        vals = {}
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                out.append(f"- {w}: {r[i]} {units[i]}")
                try:
                    vals[w] = float(r[i].replace(",", ""))
                except ValueError:
                    pass
        if "dram__bytes_read.sum" in vals:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rb = vals["dram__bytes_read.sum"] * scale.get(units[hdr.index("dram__bytes_read.sum")], 1)
            wb = vals["dram__bytes_write.sum"] * scale.get(units[hdr.index("dram__bytes_write.sum")], 1)
            tu = units[hdr.index("gpu__time_duration.sum")]
            t = vals["gpu__time_duration.sum"] * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3}.get(tu, 1e-6)
            out.append(f"- DRAM traffic per launch: {(rb + wb) / 1e6:.1f} MB; {(rb + wb) / t / 1e9:.0f} GB/s under ncu")
            traffic[k] = rb + wb
        out.append("")
    open(os.path.join(PROF, f"{tag}_ncu_full.md"), "w").write("\n".join(out) + "\n")
    tj = os.path.join(PROF, "roofline_traffic.json")
    d = json.load(open(tj)) if os.path.exists(tj) else {}
    for kname in ("k_pass_v3", "k_pass_v2", "k_pass_direct"):
        if kname in traffic:
            # the bench's dominant kernel (rbgs_pass) at the finest level of config 2
            d["cfg2_uniform256"] = traffic[kname]
            d["_source"] = f"profiles/{tag}_ncu_full.md ({kname}, level-5 launch, dram read+write bytes)"
            break
    json.dump(d, open(tj, "w"), indent=1)


if __name__ == "__main__":
    os.makedirs(PROF, exist_ok=True)
    launches()
    full()
    print(open(os.path.join(PROF, f"{tag}_launch_shares.md")).read()[:3000])
