#!/usr/bin/env bash
# Full GPU test suite + smoke + a short C2 bench (and optional env A/B).
#   gpurun -- 'bash tools/gpu_full.sh tag [VAR "v1 v2"]'
set -u
TAG=${1:-full}; VAR=${2:-}; VALS=${3:-}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log; tail -1 $OUT/smoke.log
if [ -n "$VAR" ]; then
  for r in 1 2; do for v in $VALS; do
    env $VAR=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > $OUT/b_${v}_$r.json 2>> $OUT/bench.err
    python -c "import json;d=json.load(open('$OUT/b_${v}_$r.json'));print('$VAR=$v', round(d['value'],1), d['ms_per_step'])"
  done; done
else
  timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > $OUT/b.json 2>> $OUT/bench.err
  python -c "import json;d=json.load(open('$OUT/b.json'));print(round(d['value'],1), d['ms_per_step'])"
fi
