mkdir -p gpurun_out/sw
for s in 3 4 6; do for f in 3 4; do
  r=$(timeout 300 python bench.py --steps 10 --warmup 3 --no-extras --streams $s --fine-ctas $f 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1))")
  echo "streams $s fine_ctas $f value $r" | tee -a gpurun_out/sw/sweep.txt
done; done
for w in 0 1; do
  r=$(BS_FINE_WIDE=$w timeout 300 python bench.py --steps 10 --warmup 3 --no-extras --streams 4 --fine-ctas 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1))")
  echo "streams 4 fine_ctas 3 wide $w value $r" | tee -a gpurun_out/sw/sweep.txt
done
