#!/usr/bin/env bash
# Quick perf pass on one GPU box: C2 bench line (no CPU baseline / C3 sweep),
# ncu --set full of the FineGrainedCombined render on the frame pipeline's
# super-tile lists and on the API path's 16x16 lists, their counters.
#   gpurun --timeout 1200 -- 'bash tools/gpu_perf.sh <tag> [extra bench args]'
set -u
TAG=${1:-perf}; shift || true
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-c3 "$@" > "$OUT/bench.json" 2> "$OUT/bench.err"
echo "bench rc=$?" >> "$OUT/bench.err"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_render_fine -c 1 \
  -o "$OUT/fine_super_c2" -f python tools/profile_render.py --config c2 --variant FineGrainedCombined \
  --alpha exact --reps 1 --frame-pipeline > "$OUT/ncu_super.log" 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_render_fine -c 1 \
  -o "$OUT/fine_api_c2" -f python tools/profile_render.py --config c2 --variant FineGrainedCombined \
  --alpha exact --reps 1 > "$OUT/ncu_api.log" 2>&1
python tools/ncu_counters.py --out "$OUT/ncu_counters.json" --tag "$TAG" \
  c2_FineGrainedCombined_exact_super="$OUT/fine_super_c2.ncu-rep" \
  c2_FineGrainedCombined_exact="$OUT/fine_api_c2.ncu-rep" > "$OUT/counters.log" 2>&1
tail -c 1500 "$OUT/bench.json"; cat "$OUT/counters.log"
if [ "${GW:-0}" = 1 ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_render_gw -c 1 -o "$OUT/gw_c2" -f \
    python tools/profile_render.py --config c2 --variant GaussianWise --alpha exact --reps 1 > "$OUT/ncu_gw.log" 2>&1
  python tools/ncu_counters.py --out "$OUT/ncu_counters.json" --tag "$TAG" c2_GaussianWise_exact="$OUT/gw_c2.ncu-rep" \
    >> "$OUT/counters.log" 2>&1
  tail -1 "$OUT/counters.log"
fi
