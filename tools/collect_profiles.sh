#!/usr/bin/env bash
# Copy a gpu_evidence.sh run's evidence into profiles/ (tracked), prefixed <tag>_.
#   bash tools/collect_profiles.sh <tag>
set -eu
TAG=$1
IN=gpurun_out/$TAG
P=profiles
for c in c1 c2 c4 reference; do cp "$IN/bench_$c.json" "$P/${TAG}_bench_$c.json"; done
{ echo "# ncu --metrics gpu__time_duration.sum --clock-control none over bench.py --steps 1 --warmup 3 --no-extras --batch 4 (C2 frame pipeline; per-kernel totals, serialised / cold), run $TAG"
  python tools/launches.py "$IN/launches.csv"; } > "$P/${TAG}_launches_c2.txt"
for f in fine_api_c2 fine_super_c2 fine_api_c4 fine_super_c4 gw_c2 bwd_c2 scatter_c2; do
  [ -f "$IN/$f.ncu-rep" ] && python tools/ncu_summary.py "$IN/$f.ncu-rep" > "$P/${TAG}_ncu_$f.txt"
done
cp "$IN/ncu_counters.json" "$P/ncu_counters.json"
{ tail -3 "$IN/pytest_gpu.log"; cat "$IN/smoke.log"; } > "$P/${TAG}_pytest_gpu.txt"
