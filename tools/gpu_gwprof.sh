OUT=gpurun_out/gw; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_render_gw -c 1 -o $OUT/gw2 -f \
  python tools/profile_render.py --config c2 --variant GaussianWise --alpha exact --reps 1 > $OUT/p.log 2>&1
tail -1 $OUT/p.log
