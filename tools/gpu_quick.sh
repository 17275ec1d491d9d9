#!/usr/bin/env bash
# Quick GPU check after a binning/render change: parity subset, stage times
# A/B (env VAR in "$2"), short bench.  gpurun -- 'bash tools/gpu_quick.sh tag [VAR]'
set -u
TAG=${1:-quick}; VAR=${2:-BS_SORT_CLASSIC}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider \
  -k "binning or fused or super or frame or render_exact or c4 or golden or donation" > $OUT/pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest.log; tail -3 $OUT/pytest.log
for v in 0 1; do
  env $VAR=$v TAG=$VAR=$v timeout 300 python tools/diag_stages.py c2 >> $OUT/stages.txt 2>&1
done
cat $OUT/stages.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench.json'));print(d['value'],d['ms_per_step'],d.get('stage_ms'),d.get('fwd_render_ms_per_frame'))"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python tools/profile_render.py --config c2 --variant FineGrainedCombined --alpha exact --reps 3 --frame-pipeline > $OUT/launches.log 2>&1
python tools/launches.py $OUT/launches.csv > $OUT/launches_summary.txt 2>&1; head -30 $OUT/launches_summary.txt
