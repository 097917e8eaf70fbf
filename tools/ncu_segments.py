"""Stall samples / instructions per barrier-delimited SASS segment of an ncu report (which phase
of a one-CTA multi-phase kernel costs what), with the source lines of each segment."""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]; R = rows[2:]; ix = {c: i for i, c in enumerate(h)}
def f(r, c):
    try: return float(r[ix[c]] or 0)
    except Exception: return 0.0
S = "Warp Stall Sampling (All Samples)"
tot = sum(f(r, S) for r in R)
seg = []; cur = [0.0, 0.0, None, None]
for r in R:
    cur[0] += f(r, S); cur[1] += f(r, "Instructions Executed")
    if cur[2] is None: cur[2] = r[0]
    if "BAR.SYNC" in r[1]:
        cur[3] = r[0]; seg.append(tuple(cur)); cur = [0.0, 0.0, None, None]
seg.append((cur[0], cur[1], cur[2], "end"))
print(f"total samples {tot:.0f}, instructions {sum(s[1] for s in seg):.0f}")
for s in sorted(seg, reverse=True)[:n]:
    print(f"{s[0] / tot * 100:5.1f}% samples {int(s[1]):8d} instr  {s[2]}..{s[3]}")
