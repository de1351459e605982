# round-2 checks: new full-size sampled parity (fp32, cutoff), 2-rank gloo gather, benches
T=${TAG:-r02v}
timeout 1200 python -m pytest tests/test_parity_gpu.py -x -q -k "full_size_sampled" > gpurun_out/${T}_pytest_sampled.log 2>&1; tail -3 gpurun_out/${T}_pytest_sampled.log
timeout 900 python -m pytest tests/test_multi_gpu.py -x -q > gpurun_out/${T}_pytest_multi.log 2>&1; tail -3 gpurun_out/${T}_pytest_multi.log
timeout 300 python bench.py --config C5 --dtype f32 --steps 10 --warmup 3 > gpurun_out/${T}_bench_C5_f32.json 2> gpurun_out/${T}_bench_C5_f32.err; cut -c1-300 gpurun_out/${T}_bench_C5_f32.json
timeout 300 python bench.py --config C5 --fraction 0.05 --steps 10 --warmup 3 > gpurun_out/${T}_bench_C5_cut5.json 2> gpurun_out/${T}_bench_C5_cut5.err; python -c "import json; d=json.load(open('gpurun_out/${T}_bench_C5_cut5.json')); print(d['ms_per_step'], d.get('parity_sample'), d.get('active_rate'))"
TAG=$T bash scripts/gpu_sanitize.sh
