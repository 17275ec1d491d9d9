mkdir -p gpurun_out/q1
timeout 900 python -m pytest tests -m gpu -x -q -k "binning or frame_pipeline" > gpurun_out/q1/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/q1/pytest.log
timeout 300 python bench.py --steps 200 --no-extras > gpurun_out/q1/a.json 2> gpurun_out/q1/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/q1/launches.csv python bench.py --steps 2 --warmup 3 --no-extras > /dev/null 2>&1
