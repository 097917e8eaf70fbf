"""Per-source-line stall samples / instructions of an ncu report (correlated cuda,sass view):
which lines of a kernel cost what.   python tools/ncu_lines.py rep.ncu-rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = {}
fname = None
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or not r[0].isdigit() or r[2] != "-":
        continue
    key = (fname, int(r[0]))
    st, ins = float(r[4] or 0), float(r[7] or 0)
    a = agg.setdefault(key, [0.0, 0.0, r[1].strip()[:90]])
    a[0] = max(a[0], st)   # the cuda-line row repeats per function; keep one
    a[1] = max(a[1], ins)
tot = sum(v[0] for v in agg.values()) or 1
toti = sum(v[1] for v in agg.values()) or 1
print(f"samples {tot:.0f}  warp instructions {toti:.3g}")
for (f, l), (st, ins, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{st / tot * 100:5.1f}% st {ins / toti * 100:5.1f}% in  {f}:{l:<4d} {src}")
