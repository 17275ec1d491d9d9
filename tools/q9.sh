mkdir -p gpurun_out/q9
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/q9/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/q9/pytest.log
timeout 900 python tools/training_run.py --out gpurun_out/q9/training_run.csv > gpurun_out/q9/training.log 2>&1
