# bench throughput over (--streams, --fine-ctas): bash tools/sweep_streams.sh [tag]
TAG=${1:-sw}; OUT=gpurun_out/$TAG; mkdir -p $OUT; rm -f $OUT/*
for s in 2 3 4; do for f in 2 3 4; do
  timeout 300 python bench.py --steps 300 --no-extras --no-cpu-baseline --streams $s --fine-ctas $f > $OUT/s${s}_f${f}.json 2>>$OUT/err
done; done
