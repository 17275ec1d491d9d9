"""Print key metrics of every kernel in an .ncu-rep (raw page)."""
import csv
import subprocess
import sys

WANT = ["Kernel Name", "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__cycles_active.avg",
        "sm__cycles_active.max", "smsp__inst_executed.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__t_bytes.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
STALL_PREFIX = "smsp__average_warp_latency_issue_stalled_"
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, units = r[0], r[1]
for d in r[2:]:
    print("=" * 80)
    for w in WANT:
        if w in h:
            i = h.index(w)
            print(f"{w:70s} {d[i]} {units[i]}")
    st = [(h[i][len(STALL_PREFIX):], float(d[i].replace(",", ""))) for i in range(len(h))
          if h[i].startswith(STALL_PREFIX) and h[i].endswith(".ratio") and d[i] not in ("", "n/a")]
    st.sort(key=lambda x: -x[1])
    print("top stalls:", ", ".join(f"{k}={v:.2f}" for k, v in st[:6]))
