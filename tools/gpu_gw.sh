OUT=gpurun_out/gw; mkdir -p $OUT
python -m pytest tests/test_gpu_parity.py tests/test_gpu_kat.py tests/test_gpu_configs.py -x -q -p no:cacheprovider -k "render or gaussian or Gaussian or kat or c3 or c5 or c2" 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__cycles_active.max,sm__cycles_active.avg --clock-control none --csv --log-file $OUT/gw.csv \
  python tools/profile_render.py --config c2 --variant GaussianWise --alpha exact --reps 2 > $OUT/l.log 2>&1
grep -E 'k_render_gw' $OUT/gw.csv | awk -F'","' '{print $(NF-2), $NF}' | cut -c1-150
