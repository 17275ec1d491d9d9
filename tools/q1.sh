mkdir -p gpurun_out/q1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q1/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/q1/pytest.log
for r in 1 2; do timeout 300 python bench.py --steps 200 --no-extras > gpurun_out/q1/g$r.json 2> gpurun_out/q1/bench.err; done
