mkdir -p gpurun_out/q1
timeout 900 python -m pytest tests -m gpu -x -q -k "binning" > gpurun_out/q1/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/q1/pytest.log
for wv in 1 2 4; do BS_BIN_CHUNK_WAVES=$wv timeout 300 python bench.py --no-extras --steps 100 > gpurun_out/q1/bench_w$wv.json 2> gpurun_out/q1/bench.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/q1/launches.csv python bench.py --steps 2 --warmup 3 --no-extras > /dev/null 2>&1
