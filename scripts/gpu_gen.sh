# general-span row variant: admission stats, C5 windows element by element, full-size sampled, benches
T=${TAG:-r02y}
python scripts/row_stats.py C5 C4 2>&1 | tail -2 | cut -c1-400
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "c5_regions or row_path or c1_full or c2_full or c3_full" > gpurun_out/${T}_pytest.log 2>&1; tail -3 gpurun_out/${T}_pytest.log
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "full_size_sampled" > gpurun_out/${T}_pytest_sampled.log 2>&1; tail -3 gpurun_out/${T}_pytest_sampled.log
for c in C4 C5; do
timeout 300 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
python -c "import json; d=json.load(open('gpurun_out/${T}_bench_$c.json')); print('$c', round(d['ms_per_step'],3), 'ms frac', round(d['roofline']['frac'],3), d['gpu_launches'])" || tail -3 gpurun_out/${T}_bench_$c.err
done
timeout 300 python bench.py --config C5 --dtype f32 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench_C5f32.json 2> gpurun_out/${T}_bench_C5f32.err
python -c "import json; d=json.load(open('gpurun_out/${T}_bench_C5f32.json')); print('C5 f32', round(d['ms_per_step'],3), 'ms frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/${T}_bench_C5f32.err
timeout 300 python bench.py --config C5 --noise 1 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench_C5n.json 2> gpurun_out/${T}_bench_C5n.err
python -c "import json; d=json.load(open('gpurun_out/${T}_bench_C5n.json')); print('C5 noise', round(d['ms_per_step'],3), 'ms frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/${T}_bench_C5n.err
