mkdir -p gpurun_out/q1
timeout 900 python -m pytest tests -m gpu -x -q -k "frame_pipeline or render_exact" > gpurun_out/q1/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/q1/pytest.log
for r in 1 2 3; do timeout 300 python bench.py --steps 200 --no-extras > gpurun_out/q1/d$r.json 2>> gpurun_out/q1/bench.err; done
timeout 600 python bench.py --steps 200 --no-cpu-baseline > gpurun_out/q1/full.json 2>> gpurun_out/q1/bench.err
