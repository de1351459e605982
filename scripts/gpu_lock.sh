# lock-kernel iteration: new tests first, then everything, bench C4, ncu of the lock kernel
TAG=${1:-lk}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "lock or c1_full or c2_full" 2>&1 | tail -15
timeout 300 python scripts/plan_stats.py C4 2>&1 | tail -2 | cut -c1-600
timeout 300 python bench.py --config C4 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; tail -3 gpurun_out/${TAG}_bench.err
python -c "
import json; d=json.load(open('gpurun_out/${TAG}_bench.json')); print('ms', d['ms_per_step'], 'GB/s', d['roofline']['achieved'], 'frac', d['roofline']['frac'], d.get('parity_sample'))"
DAXM_NO_LOCK=1 timeout 300 python bench.py --config C4 --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NO_LOCK ms', d['ms_per_step'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:deposit_lock -s 1 -c 1 \
   -o gpurun_out/${TAG}_lock python bench.py --config C4 --steps 1 --warmup 1 --e2e-steps 0 \
   --no-cpu-baseline > /dev/null 2> gpurun_out/${TAG}_ncu.err; tail -2 gpurun_out/${TAG}_ncu.err
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -15
