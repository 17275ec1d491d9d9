mkdir -p gpurun_out/q1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q1/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/q1/pytest.log
