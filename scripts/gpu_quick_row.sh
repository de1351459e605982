# quick A/B of the row kernel: admission stats, C4 bench, one ncu capture, CHECK-build parity on C1-C3
T=${TAG:-r02u}
python scripts/row_stats.py C2 C3 C4 2>&1 | tail -3 | cut -c1-160
timeout 120 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python -c "import json; d=json.load(open('gpurun_out/${T}_bench.json')); print('C4', round(d['ms_per_step'],3), 'ms frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/${T}_bench.err
TAG=$T bash scripts/gpu_ncu_var.sh
DAXM_LIBRARY=paper_2201_13309_b200/variants/v_check.so timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "c1 or c2 or c3 or row_path" > gpurun_out/${T}_pytest_check.log 2>&1; tail -3 gpurun_out/${T}_pytest_check.log
