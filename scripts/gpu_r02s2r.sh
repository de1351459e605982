T=${TAG:-r02s2r}
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "both or step_weights" > gpurun_out/${T}_pytest_b.log 2>&1; tail -2 gpurun_out/${T}_pytest_b.log; grep -E "^E " gpurun_out/${T}_pytest_b.log | head -5
for L in paper_2201_13309_b200/libdaxm.so; do DAXM_LIBRARY=$L timeout 300 python bench.py --config C4 --edge both --steps 5 --warmup 2 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${T}_both.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/${T}_both.json')); print('C4 both', round(d['ms_per_step'],3))"; done
NONCU=1 ROUNDS=2 TAG=$T bash scripts/gpu_ab_check.sh "$@"
