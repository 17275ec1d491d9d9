mkdir -p gpurun_out/q5
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q5/pytest.log 2>&1; echo rc=$? >> gpurun_out/q5/pytest.log
for t in a b; do
timeout 300 python bench.py --steps 200 --no-extras --no-cpu-baseline > gpurun_out/q5/fu_$t.json 2>>gpurun_out/q5/err
BS_NO_FUSED_PRE=1 timeout 300 python bench.py --steps 200 --no-extras --no-cpu-baseline > gpurun_out/q5/nofu_$t.json 2>>gpurun_out/q5/err
done
timeout 300 python bench.py --steps 50 --no-cpu-baseline > gpurun_out/q5/full.json 2>>gpurun_out/q5/err
timeout 300 python bench.py --steps 400 --no-extras --no-cpu-baseline --config c1 > gpurun_out/q5/c1.json 2>>gpurun_out/q5/err
timeout 300 python bench.py --steps 40 --no-extras --no-cpu-baseline --config c4 > gpurun_out/q5/c4.json 2>>gpurun_out/q5/err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/q5/launches.csv \
  python bench.py --steps 2 --warmup 4 --no-extras > gpurun_out/q5/launches_bench.log 2>&1
