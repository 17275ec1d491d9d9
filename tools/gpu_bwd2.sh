OUT=gpurun_out/bw; mkdir -p $OUT
python -m pytest tests/test_gpu_backward.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file $OUT/bw.csv \
  python tools/profile_render.py --config c2 --variant FineGrainedCombined --alpha exact --reps 3 --backward > $OUT/l.log 2>&1
grep -E 'k_render_backward|k_render_fine' $OUT/bw.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-150
