# full GPU record: pytest -m gpu, default bench (C4), C5 bench, launch list
T=${TAG:-r02s}
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${T}_pytest_gpu.log 2>&1; tail -5 gpurun_out/${T}_pytest_gpu.log
for c in C4 C5; do
timeout 300 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
python -c "import json; d=json.load(open('gpurun_out/${T}_bench_$c.json')); print('$c', round(d['ms_per_step'],3), 'ms frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/${T}_bench_$c.err
done
