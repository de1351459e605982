T=${TAG:-r02ze}
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "both or c1_full or c2_full or zero_skip or row_path" > gpurun_out/${T}_pytest.log 2>&1; tail -3 gpurun_out/${T}_pytest.log; grep -E "^E " gpurun_out/${T}_pytest.log | head -5
for e in leading both; do
timeout 300 python bench.py --config C4 --edge $e --steps 10 --warmup 3 --e2e-steps 0 > gpurun_out/${T}_bench_C4_$e.json 2> gpurun_out/${T}_bench_C4_$e.err
python -c "import json; d=json.load(open('gpurun_out/${T}_bench_C4_$e.json')); print('C4 $e', round(d['ms_per_step'],3), 'ms frac', round(d['roofline']['frac'],3), d['gpu_launches'], d.get('parity_sample'))" || tail -3 gpurun_out/${T}_bench_C4_$e.err
done
