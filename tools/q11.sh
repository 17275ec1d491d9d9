mkdir -p gpurun_out/q11; rm -f gpurun_out/q11/*
for kb in 40 66 132; do TAG=kb$kb BS_SC_TABLE_KB=$kb timeout 300 python tools/diag_stages.py c4 >> gpurun_out/q11/out.txt 2>&1; done
for kb in 40 66 132; do BS_SC_TABLE_KB=$kb timeout 300 python bench.py --config c4 --steps 40 --no-extras --no-cpu-baseline > gpurun_out/q11/c4_$kb.json 2>>gpurun_out/q11/err; done
