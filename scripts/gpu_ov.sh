# overlap-tile kernel: plan stats, parity on the overlap tests, C5/C4 bench, C5 launch list
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 300 python scripts/plan_stats.py C5 2>&1 | tail -1 | cut -c1-900
timeout 1200 python -m pytest tests/test_parity_gpu.py -q -x -k "overlap or C5 or lock or cutoff" 2>&1 | tail -5
CFGS="C5 C4" bash scripts/bench_all.sh
DAXM_NO_LOCK_OV=1 timeout 300 python bench.py --config C5 --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5 without the overlap lock kernel', d['ms_per_step'])"
bash scripts/gpu_launches.sh ov_C5 C5 2>&1 | tail -8
