mkdir -p gpurun_out/q5
timeout 900 python -m pytest tests -m gpu -x -q -k "render or frame" > gpurun_out/q5/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/q5/pytest.log
timeout 300 python bench.py --steps 100 --no-cpu-baseline > gpurun_out/q5/bench.json 2> gpurun_out/q5/bench.err
