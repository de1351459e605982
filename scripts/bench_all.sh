# device-resident bench of every config (no e2e / cpu baseline); prints one summary line each
mkdir -p gpurun_out/all
for c in ${CFGS:-C2 C3 C4 C5}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/all/$c.json 2> gpurun_out/all/$c.err
  python -c "import json; d=json.load(open('gpurun_out/all/$c.json')); print('$c', round(d['ms_per_step'],3), 'ms', '%.3g' % d['value'], 'px.steps/s frac', round(d['roofline']['frac'],3), 'general', d['plan']['general_tiles'], '/', d['plan']['n_tiles'])" || tail -3 gpurun_out/all/$c.err
done
