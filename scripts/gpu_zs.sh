export T=${TAG:-r02zd}
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "zero_skip or peaks_only or c5_regions or full_size_sampled or cutoff" > gpurun_out/${T}_pytest.log 2>&1; tail -3 gpurun_out/${T}_pytest.log
for c in C4 C5; do
timeout 300 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
python -c "import json; d=json.load(open('gpurun_out/${T}_bench_$c.json')); print('$c', round(d['ms_per_step'],3), 'ms frac', round(d['roofline']['frac'],3), d['gpu_launches'])" || tail -3 gpurun_out/${T}_bench_$c.err
done
DAXM_NO_ZERO_SKIP=1 timeout 300 python bench.py --config C5 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench_C5_noskip.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/${T}_bench_C5_noskip.json')); print('C5 noskip', round(d['ms_per_step'],3))"
timeout 300 python bench.py --config C5 --fraction 0.05 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench_C5_cut.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/${T}_bench_C5_cut.json')); print('C5 5%', round(d['ms_per_step'],3))"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --config C5 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/'+__import__('os').environ.get('T','r02zd')+'_launches.csv')) if len(r)>10]
hdr=rows[0]; ki=hdr.index('Kernel Name'); vi=hdr.index('Metric Value')
from collections import defaultdict
d=defaultdict(list)
for r in rows[1:]: d[r[ki][:60]].append(float(r[vi].replace(',','')))
for k,v in sorted(d.items(), key=lambda x:-sum(x[1])): print(f"{k:60s} n={len(v)} mean_us={sum(v)/len(v)/1e3:.1f}")
PY
