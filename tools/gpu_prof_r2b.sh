#!/usr/bin/env bash
# r2b: source-level ncu captures of the hot kernels (FG api/super C2, GW C2,
# scatter + radix scatter in the frame pipeline) and the frame-pipeline
# launch list; .ncu-rep files come back in gpurun_out/<tag>/.
set -u
TAG=${1:-r2b}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_render_fine -c 1 \
  -o "$OUT/fine_api_c2" -f python tools/profile_render.py --config c2 --variant FineGrainedCombined \
  --alpha exact --reps 1 > "$OUT/ncu_api.log" 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_render_fine -c 1 \
  -o "$OUT/fine_super_c2" -f python tools/profile_render.py --config c2 --variant FineGrainedCombined \
  --alpha exact --reps 1 --frame-pipeline > "$OUT/ncu_super.log" 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_render_gw -c 1 -o "$OUT/gw_c2" -f \
  python tools/profile_render.py --config c2 --variant GaussianWise --alpha exact --reps 1 > "$OUT/ncu_gw.log" 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_chunk_scatter|k_radix|k_project_bin|k_chunk_hist|k_scan" -c 12 \
  -o "$OUT/bin_c2" -f python tools/profile_render.py --config c2 --variant FineGrainedCombined \
  --alpha exact --reps 1 --frame-pipeline > "$OUT/ncu_bin.log" 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
  python tools/profile_render.py --config c2 --variant FineGrainedCombined --alpha exact --reps 3 --frame-pipeline > "$OUT/launches.log" 2>&1
python tools/launches.py "$OUT/launches.csv" > "$OUT/launches_summary.txt" 2>&1
echo done
