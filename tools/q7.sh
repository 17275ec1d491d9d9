mkdir -p gpurun_out/q7
timeout 1200 python -m pytest tests -m gpu -x -q -k "c4_tile_sampled" > gpurun_out/q7/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/q7/pytest.log
timeout 600 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/q7/bench_c4.json 2> gpurun_out/q7/bench_c4.err
timeout 600 python bench.py --config c1 --steps 200 --no-cpu-baseline > gpurun_out/q7/bench_c1.json 2> gpurun_out/q7/bench_c1.err
timeout 900 python tools/sweep_c3.py --out gpurun_out/q7/c3_sweep.jsonl > gpurun_out/q7/c3.log 2>&1
