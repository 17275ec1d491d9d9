#!/usr/bin/env bash
# Copy a gpu_round.sh run's evidence into profiles/ (tracked).
#   bash tools/collect_profiles.sh <tag>
set -eu
IN=gpurun_out/$1
P=profiles
cp "$IN/bench.json" $P/r1_bench_c2.json
cp "$IN/bench_c1.json" $P/r1_bench_c1.json
cp "$IN/bench_c4.json" $P/r1_bench_c4.json
cp "$IN/bench_reference.json" $P/r1_bench_reference.json
python tools/launches.py "$IN/launches.csv" > $P/r1_launches_c2.txt
python tools/ncu_summary.py "$IN/render_fine_full.ncu-rep" > $P/r1_ncu_full_render_fine_exact.txt
for c in c1 c4; do
  [ -f "$IN/render_fine_full_$c.ncu-rep" ] && \
    python tools/ncu_summary.py "$IN/render_fine_full_$c.ncu-rep" > $P/r1_ncu_full_render_fine_exact_$c.txt
done
for c in c2 c4; do
  [ -f "$IN/render_fine_super_$c.ncu-rep" ] && \
    python tools/ncu_summary.py "$IN/render_fine_super_$c.ncu-rep" > $P/r1_ncu_full_render_fine_super_$c.txt
done
python tools/ncu_traffic.py $P > $P/ncu_traffic.json
python tools/ncu_summary.py "$IN/chunk_scatter_full.ncu-rep" > $P/r1_ncu_chunk_scatter.txt
cp "$IN/c3_sweep.jsonl" $P/r1_c3_sweep.jsonl
cp "$IN/training_run.csv" $P/r1_training_run.csv
{ tail -3 "$IN/pytest_gpu.log"; cat "$IN/smoke.log"; } > $P/r1_pytest_gpu.txt
grep -m1 "Model name" "$IN/nproc.txt" > $P/r1_host.txt || true
head -1 "$IN/nproc.txt" >> $P/r1_host.txt
