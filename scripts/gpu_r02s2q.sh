T=${TAG:-r02s2q}
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "step_weights or out_of_core or general_wire or graph" > gpurun_out/${T}_pytest_w.log 2>&1; tail -2 gpurun_out/${T}_pytest_w.log; grep -E "^E " gpurun_out/${T}_pytest_w.log | head -5
timeout 300 python scripts/row_stats.py C2 C3 C4 C5 C2:trailing 2>&1 | tail -5 | cut -c1-330
NONCU=1 ROUNDS=2 TAG=$T bash scripts/gpu_ab_check.sh "$@"
