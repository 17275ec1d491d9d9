mkdir -p gpurun_out/q1
timeout 900 python -m pytest tests -m gpu -x -q -k "binning or frame_pipeline" > gpurun_out/q1/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/q1/pytest.log
for wv in 1 2 4; do BS_BIN_CHUNK_WAVES=$wv timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_chunk --csv --log-file gpurun_out/q1/w$wv.csv python tools/profile_render.py --reps 3 > /dev/null 2>&1; done
