#!/usr/bin/env bash
# Full evidence pass on one B200: GPU tests, smoke, the C2 bench line
# (defaults: batch step, extras incl. C3 sweep / e2e / cpu_baseline), C1 and
# C4 lines, the reference arm (complete frames), a launch list, ncu counters
# of the render kernels.  Outputs in gpurun_out/<tag>/.
#   gpurun --timeout 3600 -- 'bash tools/gpu_evidence.sh <tag>'
set -u
TAG=${1:-r2}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
nproc > "$OUT/nproc.txt"; lscpu >> "$OUT/nproc.txt" 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
tail -3 "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
timeout 900 python bench.py --steps 20 --warmup 5 > "$OUT/bench_c2.json" 2> "$OUT/bench.err"; echo "bench rc=$?" >> "$OUT/bench.err"
timeout 600 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu-baseline --no-c3 > "$OUT/bench_c1.json" 2>> "$OUT/bench.err"
timeout 900 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-c3 > "$OUT/bench_c4.json" 2>> "$OUT/bench.err"
timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 > "$OUT/bench_reference.json" 2>> "$OUT/bench.err"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
  python bench.py --steps 1 --warmup 3 --no-extras --batch 4 > "$OUT/launches_bench.log" 2>&1
python tools/launches.py "$OUT/launches.csv" > "$OUT/launches_summary.txt" 2>&1
for c in c2 c4; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_render_fine -c 1 \
    -o "$OUT/fine_super_$c" -f python tools/profile_render.py --config $c --variant FineGrainedCombined \
    --alpha exact --reps 1 --frame-pipeline > "$OUT/ncu_super_$c.log" 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_render_fine -c 1 \
    -o "$OUT/fine_api_$c" -f python tools/profile_render.py --config $c --variant FineGrainedCombined \
    --alpha exact --reps 1 > "$OUT/ncu_api_$c.log" 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_render_gw -c 1 -o "$OUT/gw_c2" -f \
  python tools/profile_render.py --config c2 --variant GaussianWise --alpha exact --reps 1 > "$OUT/ncu_gw.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_render_backward -c 1 -o "$OUT/bwd_c2" -f \
  python tools/profile_render.py --config c2 --variant FineGrainedCombined --alpha exact --reps 1 --backward > "$OUT/ncu_bwd.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chunk_scatter -c 1 -o "$OUT/scatter_c2" -f \
  python tools/profile_render.py --config c2 --variant FineGrainedCombined --alpha exact --reps 1 --frame-pipeline \
  > "$OUT/ncu_scatter.log" 2>&1
python tools/ncu_counters.py --out "$OUT/ncu_counters.json" --tag "$TAG" \
  c2_FineGrainedCombined_exact_super="$OUT/fine_super_c2.ncu-rep" c2_FineGrainedCombined_exact="$OUT/fine_api_c2.ncu-rep" \
  c4_FineGrainedCombined_exact_super="$OUT/fine_super_c4.ncu-rep" c4_FineGrainedCombined_exact="$OUT/fine_api_c4.ncu-rep" \
  c2_GaussianWise_exact="$OUT/gw_c2.ncu-rep" c2_chunk_scatter_super="$OUT/scatter_c2.ncu-rep" \
  c2_backward_exact="$OUT/bwd_c2.ncu-rep" > "$OUT/counters.log" 2>&1
echo done
