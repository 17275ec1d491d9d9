mkdir -p gpurun_out/q1
for ns in 1 2 3; do timeout 300 python bench.py --steps 200 --no-extras --streams $ns > gpurun_out/q1/s$ns.json 2>> gpurun_out/q1/bench.err; done
for ns in 1 2 3; do BS_CLOCKS=off timeout 300 python bench.py --steps 200 --no-extras --streams $ns > gpurun_out/q1/off$ns.json 2>> gpurun_out/q1/bench.err; done
python tools/diag_dual.py > gpurun_out/q1/dual.txt 2>&1
FLUSH=1 python tools/diag_dual.py > gpurun_out/q1/dual_flush.txt 2>&1
