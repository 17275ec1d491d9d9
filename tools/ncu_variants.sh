#!/usr/bin/env bash
# ncu --set full of every render variant's kernel(s) on C2 and C4,
# one frame each (bench's first view, exact alpha).  Outputs under
# gpurun_out/<tag>/variants/; tools/ncu_summary.py turns each into text.
#   gpurun --timeout 1800 -- 'bash tools/ncu_variants.sh r1v'
set -u
OUT=gpurun_out/${1:-r1v}/variants
mkdir -p "$OUT"
for c in c2 c4; do
  for v in Naive DynamicBlocks SharedMemOpt GaussianWise FineGrainedCombined; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_render_ -c 2 \
      -o "$OUT/${c}_$v" -f python tools/profile_render.py --config $c --variant $v --alpha exact --reps 1 \
      > "$OUT/${c}_$v.log" 2>&1
    echo "$c $v rc=$?" >> "$OUT/status.txt"
  done
done
