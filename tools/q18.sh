OUT=gpurun_out/q18; mkdir -p $OUT; rm -f $OUT/*
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
BS_SUPER_RECT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "frame or c4 or views" > $OUT/pytest_rect.log 2>&1; echo rc=$? >> $OUT/pytest_rect.log
for cfg in "BS_NO_SUPER=1" "BS_SUPER_RECT=0" "BS_SUPER_RECT=1"; do
  env $cfg TAG=$cfg timeout 300 python tools/diag_stages.py c2 >> $OUT/stages.txt 2>&1
  env $cfg TAG=$cfg timeout 300 python tools/diag_stages.py c4 >> $OUT/stages.txt 2>&1
  env $cfg timeout 300 python bench.py --steps 200 --no-extras --no-cpu-baseline > $OUT/b_$cfg.json 2>>$OUT/err
  env $cfg timeout 300 python bench.py --steps 30 --no-extras --no-cpu-baseline --config c4 > $OUT/c4_$cfg.json 2>>$OUT/err
done
