"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per-kernel totals of the last step."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
data = rows[hi + 1:]
last = int(sys.argv[2]) if len(sys.argv) > 2 else len(data)
tot = collections.OrderedDict()
cnt = collections.Counter()
for r in data[-last:]:
    name = r[ki].split("(")[0][:64]
    tot[name] = tot.get(name, 0) + float(r[vi].replace(",", ""))
    cnt[name] += 1
s = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v / 1e3:9.1f} us  {v / s * 100:5.1f}%  x{cnt[k]:<3d} {k}")
print(f"total {s / 1e3:.1f} us over {sum(cnt.values())} launches")
