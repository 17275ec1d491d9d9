#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py
#   gpurun --timeout 2400 -- 'bash tools/sanitize.sh <tag>'
set -u
TAG=${1:-san}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
for tool in memcheck racecheck synccheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check full"
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --log-file "$OUT/$tool.log" \
    python tools/sanitize_run.py > "$OUT/$tool.out" 2>&1
  echo "$tool rc=$?" >> "$OUT/summary.txt"
  tail -3 "$OUT/$tool.log" >> "$OUT/summary.txt"
done
cat "$OUT/summary.txt"
