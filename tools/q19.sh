OUT=gpurun_out/q19; mkdir -p $OUT; rm -f $OUT/*
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for cfg in "BS_NO_SUPER=1" "BS_NO_SUPER=0"; do
  env $cfg timeout 300 python bench.py --steps 200 --no-extras --no-cpu-baseline > $OUT/b_$cfg.json 2>>$OUT/err
  env $cfg timeout 300 python bench.py --steps 400 --no-extras --no-cpu-baseline --config c1 > $OUT/c1_$cfg.json 2>>$OUT/err
  env $cfg timeout 300 python bench.py --steps 30 --no-extras --no-cpu-baseline --config c4 > $OUT/c4_$cfg.json 2>>$OUT/err
done
timeout 600 python bench.py --steps 100 --no-cpu-baseline > $OUT/full.json 2>>$OUT/err
