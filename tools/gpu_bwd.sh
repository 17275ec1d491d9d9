OUT=gpurun_out/bw; mkdir -p $OUT
timeout 900 python bench.py --steps 5 --warmup 3 --no-c3 --no-cpu-baseline > $OUT/b.json 2> $OUT/b.err
python -c "import json;d=json.load(open('$OUT/b.json'));print(d['value'], d.get('bwd_render_ms_per_frame'), d['render_ms_by_variant']['exact'], d.get('e2e',{}).get('value'))"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_render_backward -c 1 -o $OUT/bwd_c2 -f \
  python tools/profile_render.py --config c2 --variant FineGrainedCombined --alpha exact --reps 1 --backward > $OUT/ncu.log 2>&1
tail -2 $OUT/ncu.log
