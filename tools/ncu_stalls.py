"""Stall-reason breakdown (pc sampling) per kernel of an .ncu-rep."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
for d in r[2:]:
    name = d[h.index("Kernel Name")][:60]
    tot = {}
    for i, k in enumerate(h):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            try:
                tot[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(d[i].replace(",", ""))
            except ValueError:
                pass
    s = sum(tot.values()) or 1
    top = sorted(tot.items(), key=lambda x: -x[1])[:8]
    print(name, "|", ", ".join(f"{k} {v / s * 100:.0f}%" for k, v in top))
