OUT=gpurun_out/q17; mkdir -p $OUT; rm -f $OUT/*
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for v in 0 1; do
  TAG=nosuper$v BS_NO_SUPER=$v timeout 300 python tools/diag_stages.py c2 >> $OUT/stages.txt 2>&1
  TAG=nosuper$v BS_NO_SUPER=$v timeout 300 python tools/diag_stages.py c4 >> $OUT/stages.txt 2>&1
  BS_NO_SUPER=$v timeout 300 python bench.py --steps 200 --no-extras --no-cpu-baseline > $OUT/b$v.json 2>>$OUT/err
  BS_NO_SUPER=$v timeout 300 python bench.py --steps 30 --no-extras --no-cpu-baseline --config c4 > $OUT/c4_$v.json 2>>$OUT/err
done
