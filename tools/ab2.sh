# A/B of two builds: bash tools/ab2.sh <tag>  (expects build_a/ and build_b/ .so sets)
TAG=${1:-ab}; OUT=gpurun_out/$TAG; mkdir -p $OUT; rm -f $OUT/*
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "binning or fused or c4 or frame" > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for r in 1 2; do
  TAG=new timeout 300 python tools/diag_stages.py c2 >> $OUT/stages.txt 2>&1
  TAG=new timeout 300 python tools/diag_stages.py c4 >> $OUT/stages.txt 2>&1
  timeout 300 python bench.py --steps 200 --no-extras --no-cpu-baseline > $OUT/b_$r.json 2>>$OUT/err
done
