#!/usr/bin/env bash
# Bench A/B of library builds (kernel-code variants): each ab_libs/<name>.so is
# copied over the in-tree library in turn, then the FG render timing
# (diag_render_time.py) and a short C2 bench run; optional pytest args run
# against the LAST build listed.  Summary in gpurun_out/<tag>/ab.txt.
#   gpurun -- 'bash tools/gpu_ab_lib.sh tag "base cand" [pytest args...]'
TAG=$1; NAMES=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
LIB=paper_2412_17378_b200/lib/libsplatsim_b200.so
for r in 1 2; do for v in $NAMES; do
  cp ab_libs/$v.so $LIB
  echo "$v render: $(timeout 300 python tools/diag_render_time.py 2>> $OUT/err.log | tail -2 | tr "\n" " ")" >> $OUT/ab.txt
  timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > $OUT/b_${v}_$r.json 2>> $OUT/err.log
  python - "$OUT/b_${v}_$r.json" "$v" >> $OUT/ab.txt <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
print(sys.argv[2], "bench:", round(d["value"], 1), "views/s", round(d["ms_per_step"], 3), "ms/step")
PY
done; done
if [ $# -gt 0 ]; then
  timeout 1500 python -m pytest -x -q -p no:cacheprovider "$@" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
  tail -2 $OUT/pytest.log >> $OUT/ab.txt
fi
cat $OUT/ab.txt
