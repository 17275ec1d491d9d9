mkdir -p gpurun_out/q1
for lg in 18 17 16; do
BS_BIN_CHUNK_LOG2=$lg timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_chunk --csv --log-file gpurun_out/q1/c4_$lg.csv python tools/profile_render.py --variant FineGrainedCombined --n 3000000 --W 3840 --H 2160 --f 2000 --reps 2 > /dev/null 2>&1
BS_BIN_CHUNK_LOG2=$lg timeout 300 python bench.py --steps 200 --no-extras > gpurun_out/q1/c2_$lg.json 2>> gpurun_out/q1/bench.err
done
