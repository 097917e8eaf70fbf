"""Summarise an ncu report's SASS source page: top instructions by L2 sectors / stalls."""
import csv, io, subprocess, sys
rep = sys.argv[1]
key = sys.argv[2] if len(sys.argv) > 2 else "L2 Theoretical Sectors Global"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]; R = rows[2:]
ix = {c: i for i, c in enumerate(h)}
def f(r, c):
    try: return float(r[ix[c]] or 0)
    except Exception: return 0.0
for c in ["L2 Theoretical Sectors Global", "L2 Theoretical Sectors Global Excessive", "L1 Wavefronts Shared",
          "L1 Wavefronts Shared Excessive", "Warp Stall Sampling (All Samples)", "Instructions Executed"]:
    print(f"{c}: {sum(f(r, c) for r in R):.4g}")
print(f"instructions: {len(R)}")
for r in sorted(R, key=lambda r: -f(r, key))[:n]:
    print(r[0][-5:], r[1].strip()[:70].ljust(70), int(f(r, "Instructions Executed")), round(f(r, "Avg. Threads Executed"), 1),
          int(f(r, "L2 Theoretical Sectors Global")), int(f(r, "L1 Wavefronts Shared")), int(f(r, "Warp Stall Sampling (All Samples)")))
