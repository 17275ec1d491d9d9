bash tools/gpu_full.sh f2
bash tools/sanitize.sh san2 > /dev/null 2>&1; cat gpurun_out/san2/summary.txt
