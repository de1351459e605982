mkdir -p gpurun_out
for v in variants/*.so; do
  r=$(DAXM_LIBRARY=$v timeout 300 python bench.py --config ${CFG:-C4} --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d.get('parity_sample',{}).get('pass'))")
  echo "$v $r"
done
