mkdir -p gpurun_out/q7
timeout 1200 python -m pytest tests -m gpu -x -q -k "c4_tile_sampled or binning" > gpurun_out/q7/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/q7/pytest.log
timeout 600 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/q7/bench_c4.json 2> gpurun_out/q7/bench_c4.err
timeout 600 python bench.py --steps 200 --no-extras > gpurun_out/q7/bench_c2.json 2> gpurun_out/q7/bench_c2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/q7/c4.csv python tools/profile_render.py --variant FineGrainedCombined --n 3000000 --W 3840 --H 2160 --f 2000 --reps 2 > /dev/null 2>&1
