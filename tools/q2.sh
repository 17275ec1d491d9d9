set -u
mkdir -p gpurun_out/q2
uptime > gpurun_out/q2/info.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "render_views or graph_replay or torch_stream" > gpurun_out/q2/pytest.log 2>&1; echo rc=$? >> gpurun_out/q2/pytest.log
for t in a b; do timeout 300 python bench.py --steps 200 --no-extras > gpurun_out/q2/d$t.json 2>>gpurun_out/q2/err; done
timeout 300 python bench.py --steps 200 --no-extras --streams 1 > gpurun_out/q2/s1.json 2>>gpurun_out/q2/err
timeout 300 python bench.py --steps 200 --no-extras --streams 2 > gpurun_out/q2/s2.json 2>>gpurun_out/q2/err
timeout 300 python bench.py --steps 400 --no-extras --config c1 > gpurun_out/q2/c1.json 2>>gpurun_out/q2/err
timeout 300 python bench.py --steps 40 --no-extras --config c4 > gpurun_out/q2/c4.json 2>>gpurun_out/q2/err
