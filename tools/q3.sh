OUT=gpurun_out/r1h
mkdir -p $OUT
for c in c1 c4; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_render_fine -c 1 \
    -o "$OUT/render_fine_full_$c" -f python tools/profile_render.py --config $c --variant FineGrainedCombined \
    --alpha exact --reps 1 > "$OUT/ncu_full_$c.log" 2>&1
done
