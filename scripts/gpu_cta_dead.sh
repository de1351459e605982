# usage: bash scripts/gpu_cta_dead.sh -- cutoff tests + C5 5 %/50 % and C4 benches (CTA-level dead-group exit A/B)
mkdir -p gpurun_out/cta
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "cutoff or sparse" 2>&1 | tail -2
for rep in 1 2; do
  for f in 0.05 0.5; do
    timeout 600 python bench.py --config C5 --fraction $f --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/cta/C5_f${f}_$rep.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/cta/C5_f${f}_$rep.json')); print('C5 f$f rep $rep', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms_median'],3))"
  done
  timeout 600 python bench.py --config C4 --steps 20 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/cta/C4_$rep.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/cta/C4_$rep.json')); print('C4 rep $rep', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms_median'],3))"
done
