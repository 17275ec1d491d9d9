"""Per-kernel measured counters from ncu --set full captures -> profiles/ncu_counters.json
(bench.py's roofline picks its bound from these and reports them).

  python tools/ncu_counters.py --out profiles/ncu_counters.json KEY=path.ncu-rep [KEY=path.ncu-rep ...]

KEY is "<config>_<Variant>_<mode>[_super]" (e.g. c2_FineGrainedCombined_exact_super).
For each report the FIRST launch of the captured kernel is read through
`ncu -i <rep> --page raw --csv`; existing keys in --out are kept unless
overwritten.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess

METRICS = {
    "duration_ns": "gpu__time_duration.sum",
    "inst_executed": "smsp__inst_executed.sum",
    "avg_active_lanes": "smsp__thread_inst_executed_per_inst_executed.ratio",
    "avg_pred_on_lanes": "smsp__thread_inst_executed_pred_on_per_inst_executed.ratio",
    "warps_active_per_smsp": "smsp__warps_active.avg.per_cycle_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "warp_exec_efficiency_pct": "smsp__thread_inst_executed_per_inst_executed.pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6,
         "second": 1e9, "inst": 1, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9, "%": 1, "": 1}


def read(rep: str) -> dict:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    head, units, first = rows[0], rows[1], rows[2]
    col = {name: i for i, name in enumerate(head)}
    out = {"kernel": first[col["Kernel Name"]][:120] if "Kernel Name" in col else None}
    for key, m in METRICS.items():
        if m in col:
            v = first[col[m]].replace(",", "")
            try:
                out[key] = float(v) * SCALE.get(units[col[m]], 1)
            except ValueError:
                pass
    if "dram_read" in out and "dram_write" in out:
        out["dram_bytes"] = int(out["dram_read"] + out["dram_write"])
    if "inst_executed" in out:
        out["inst_executed"] = int(out["inst_executed"])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--tag", default="")
    ap.add_argument("pairs", nargs="+")
    a = ap.parse_args()
    data = {}
    if os.path.exists(a.out):
        with open(a.out) as f:
            data = json.load(f)
    for p in a.pairs:
        key, path = p.split("=", 1)
        d = read(path)
        d["source"] = f"{os.path.basename(path)} ({a.tag}): ncu --set full --clock-control none, first launch, cold"
        data[key] = d
        print(key, json.dumps(d))
    with open(a.out, "w") as f:
        json.dump(data, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
