T=${TAG:-r02w}
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_multi_gpu.py -x -q -k "sharded or two_ranks or c1_full or row_path" > gpurun_out/${T}_pytest.log 2>&1; tail -3 gpurun_out/${T}_pytest.log
timeout 120 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python -c "import json; d=json.load(open('gpurun_out/${T}_bench.json')); print('C4', round(d['ms_per_step'],3), 'ms frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/${T}_bench.err
CS="compute-sanitizer --print-limit 50 --error-exitcode 9"
timeout 900 $CS --tool memcheck --leak-check full python scripts/sanitize_case.py > gpurun_out/${T}_san_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -2 gpurun_out/${T}_san_memcheck.log
timeout 1200 $CS --tool racecheck --racecheck-report analysis python scripts/sanitize_case.py c1 c1p ragged general cut > gpurun_out/${T}_san_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -2 gpurun_out/${T}_san_racecheck.log
