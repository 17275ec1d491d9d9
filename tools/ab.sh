# A/B of an env knob on the GPU box: bash tools/ab.sh VAR "v1 v2 ..." [tag]
VAR=$1; VALS=$2; TAG=${3:-ab}
OUT=gpurun_out/$TAG; mkdir -p $OUT; rm -f $OUT/*
env $VAR=${VALS%% *} timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "binning or fused or c4 or frame" > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for r in 1 2; do for v in $VALS; do
  env $VAR=$v TAG=$v timeout 300 python tools/diag_stages.py c2 >> $OUT/stages.txt 2>&1
  env $VAR=$v TAG=$v timeout 300 python tools/diag_stages.py c4 >> $OUT/stages.txt 2>&1
  env $VAR=$v timeout 300 python bench.py --steps 200 --no-extras --no-cpu-baseline > $OUT/b_${v}_$r.json 2>>$OUT/err
done; done
