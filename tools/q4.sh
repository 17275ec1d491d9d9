mkdir -p gpurun_out/q4
timeout 300 python bench.py --steps 100 --no-cpu-baseline --no-extras > gpurun_out/q4/lpt.json 2> gpurun_out/q4/err
BS_FINE_NO_LPT=1 timeout 300 python bench.py --steps 100 --no-cpu-baseline --no-extras > gpurun_out/q4/nolpt.json 2>> gpurun_out/q4/err
for s in 0.035 0.02 0.012; do
python tools/profile_render.py --reps 1 > /dev/null 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_render --csv --log-file gpurun_out/q4/lpt.csv python tools/profile_render.py --variant FineGrainedCombined --sigma 0.012 --reps 2 > /dev/null 2>&1
BS_FINE_NO_LPT=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_render --csv --log-file gpurun_out/q4/nolpt.csv python tools/profile_render.py --variant FineGrainedCombined --sigma 0.012 --reps 2 > /dev/null 2>&1
