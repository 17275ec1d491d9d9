mkdir -p gpurun_out/q1
uptime > gpurun_out/q1/uptime.txt; nvidia-smi --query-gpu=index,name,pci.bus_id,clocks.sm,clocks.mem,power.draw,temperature.gpu --format=csv >> gpurun_out/q1/uptime.txt
for r in 1 2; do timeout 300 python bench.py --steps 200 --no-extras > gpurun_out/q1/d$r.json 2>> gpurun_out/q1/bench.err; done
timeout 300 python bench.py --steps 200 --no-extras --streams 1 > gpurun_out/q1/s1.json 2>> gpurun_out/q1/bench.err
timeout 300 python bench.py --steps 200 --no-extras --config c1 > gpurun_out/q1/c1.json 2>> gpurun_out/q1/bench.err
python tools/diag_dual.py > gpurun_out/q1/dual.txt 2>&1
top -b -n 1 | head -15 >> gpurun_out/q1/uptime.txt
