mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for rep in 1 2 3; do
  timeout 600 python bench.py --config C4 --steps 20 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab/C4_$rep.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab/C4_$rep.json')); print('C4 rep $rep', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms_median'],3))"
done
for rep in 1 2; do for n in 1 2 8; do
  DAXM_ZERO_PER_SM=$n timeout 600 python bench.py --config C5 --fraction 0.05 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab/C5_z${n}_$rep.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab/C5_z${n}_$rep.json')); print('C5 f0.05 z$n rep $rep', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms_median'],3))"
done; done
