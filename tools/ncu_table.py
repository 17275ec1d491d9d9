"""One table over several .ncu-rep files: per kernel launch, duration, DRAM
traffic, issue / warp activity and the busiest pipes.

  python tools/ncu_table.py gpurun_out/r1v/variants/*.ncu-rep > profiles/r1_ncu_variants.txt
"""
import csv
import os
import subprocess
import sys

COLS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
        ("launch__registers_per_thread", "regs"),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64%"),
        ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma%"),
        ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu%"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu%"),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%"),
        ("dram__cycles_active.avg.pct_of_peak_sustained_elapsed", "dram%")]
SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "us": 1.0, "ms": 1e3, "ns": 1e-3,
         "usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3}


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    if len(r) < 3:
        return
    h, units = r[0], r[1]
    for d in r[2:]:
        vals = []
        for key, _ in COLS:
            if key not in h:
                vals.append("-")
                continue
            i = h.index(key)
            v = float(d[i].replace(",", "")) if d[i] not in ("", "n/a") else float("nan")
            v *= SCALE.get(units[i], 1.0)
            vals.append(f"{v:.1f}")
        yield d[h.index("Kernel Name")].split("(")[0].replace("void ", ""), vals


print("# per launch; time in us, DRAM in MB (cold cache, ncu --set full, clock-control none)")
print(f"{'capture':32s} {'kernel':34s} " + " ".join(f"{n:>8s}" for _, n in COLS))
for p in sys.argv[1:]:
    for name, vals in rows(p):
        print(f"{os.path.basename(p).replace('.ncu-rep', ''):32s} {name[:34]:34s} " + " ".join(f"{v:>8s}" for v in vals))
