"""Top SASS instructions of one kernel in an .ncu-rep by stall samples and executions.
  python tools/ncu_sass_hot.py rep.ncu-rep [N]"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
r = list(csv.reader(out[1:]))
h = r[0]
rows = r[1:]
si, ei, ti = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
tot_s = sum(float(x[si] or 0) for x in rows)
tot_e = sum(float(x[ei] or 0) for x in rows)
print(f"total samples {tot_s:.0f}, warp instructions {tot_e:.0f}")
for i, x in enumerate(rows):
    s, e = float(x[si] or 0), float(x[ei] or 0)
    if s / tot_s > 0.004 or (sys.argv[3:] and e > 0):
        print(f"{i:5d} {s / tot_s * 100:5.1f}% {e:12.0f}  {x[ti].strip()[:70]}")
