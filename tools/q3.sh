mkdir -p gpurun_out/q3
for ab in 0 1 2; do BS_SC_ABLATE=$ab timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_chunk_scatter --csv --log-file gpurun_out/q3/ab$ab.csv python tools/profile_render.py --reps 3 > /dev/null 2>&1; done
