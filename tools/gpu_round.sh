#!/usr/bin/env bash
# One GPU-box pass: parity tests, smoke, bench lines (C2 headline with extras,
# C1, C4, reference arm), launch list, ncu --set full captures of the two top
# kernels, the C3 sweep and the measured training run.  Outputs land in
# gpurun_out/<tag>/ (merged back); tools/collect_profiles.sh copies the
# summaries into profiles/.
#   gpurun --timeout 3600 -- 'bash tools/gpu_round.sh [tag]'
set -u
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
nproc > "$OUT/nproc.txt"; lscpu >> "$OUT/nproc.txt" 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?" >> "$OUT/bench.err"
timeout 600 python bench.py --config c1 --no-cpu-baseline > "$OUT/bench_c1.json" 2>> "$OUT/bench.err"
timeout 900 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline > "$OUT/bench_c4.json" 2>> "$OUT/bench.err"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > "$OUT/bench_reference.json" 2>> "$OUT/bench.err"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
  python bench.py --steps 2 --warmup 4 --no-extras > "$OUT/launches_bench.log" 2>&1
for c in c2 c4; do  # the frame pipeline's render (super-tile lists at >= 1 Mpixel)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_render_fine -c 1 \
    -o "$OUT/render_fine_super_$c" -f python tools/profile_render.py --config $c --variant FineGrainedCombined \
    --alpha exact --reps 1 --frame-pipeline > "$OUT/ncu_super_$c.log" 2>&1
done
for c in c2 c1 c4; do
  sfx=$([ $c = c2 ] && echo "" || echo "_$c")
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_render_fine -c 1 \
    -o "$OUT/render_fine_full$sfx" -f python tools/profile_render.py --config $c --variant FineGrainedCombined \
    --alpha exact --reps 1 > "$OUT/ncu_full$sfx.log" 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chunk_scatter -c 1 \
  -o "$OUT/chunk_scatter_full" -f python tools/profile_render.py --variant FineGrainedCombined --alpha exact --reps 1 \
  > "$OUT/ncu_full2.log" 2>&1
timeout 1200 python tools/sweep_c3.py --out "$OUT/c3_sweep.jsonl" > "$OUT/c3.log" 2>&1
timeout 1200 python tools/training_run.py --out "$OUT/training_run.csv" > "$OUT/training.log" 2>&1
echo done
