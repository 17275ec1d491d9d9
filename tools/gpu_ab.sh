#!/usr/bin/env bash
# Bench A/B of an env knob (no tests): gpurun -- 'bash tools/gpu_ab.sh tag VAR "v1 v2 ..." [bench args]'
TAG=$1; VAR=$2; VALS=$3; shift 3
OUT=gpurun_out/$TAG; mkdir -p $OUT
for r in 1 2; do for v in $VALS; do
  env $VAR=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline "$@" > $OUT/b_${v}_$r.json 2>> $OUT/bench.err
  python -c "import json;d=json.load(open('$OUT/b_${v}_$r.json'));print('$VAR=$v', round(d['value'],1), d['ms_per_step'])"
done; done
