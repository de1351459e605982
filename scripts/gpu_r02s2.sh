# session-2 baseline: full GPU suite, C4/C5 bench, one full ncu capture of the C4 row kernel
T=${TAG:-r02s2a}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest_gpu.log 2>&1; tail -3 gpurun_out/${T}_pytest_gpu.log; grep -E "^E |FAILED" gpurun_out/${T}_pytest_gpu.log | head -8
timeout 180 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench_C4.json 2> gpurun_out/${T}_bench_C4.err; python -c "import json; d=json.load(open('gpurun_out/${T}_bench_C4.json')); print('C4', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))" || tail -3 gpurun_out/${T}_bench_C4.err
TAG=${T} bash scripts/gpu_ncu_var.sh
