#!/usr/bin/env bash
# One GPU-box pass: parity tests, smoke, bench line, launch list, one ncu --set full
# capture of the top render kernel.  Outputs land in gpurun_out/ (merged back).
#   gpurun --timeout 1800 -- 'bash tools/gpu_round.sh [tag]'
set -u
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
nproc > "$OUT/nproc.txt"; lscpu >> "$OUT/nproc.txt" 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
timeout 600 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?" >> "$OUT/bench.err"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
  python bench.py --steps 2 --warmup 3 --no-extras > "$OUT/launches_bench.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_render_fine -c 1 \
  -o "$OUT/render_fine_full" -f python tools/profile_render.py --variant FineGrainedCombined --alpha exact --reps 1 \
  > "$OUT/ncu_full.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chunk_scatter -c 1 \
  -o "$OUT/chunk_scatter_full" -f python tools/profile_render.py --variant FineGrainedCombined --alpha exact --reps 1 \
  > "$OUT/ncu_full2.log" 2>&1
echo done
