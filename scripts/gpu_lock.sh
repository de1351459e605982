# lock-kernel iteration: smoke + lock tests first, bench every config, ncu of the C4 lock kernel, full GPU suite
TAG=${1:-lk}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "lock or c1_full or c2_full" 2>&1 | tail -15
timeout 300 python scripts/plan_stats.py C4 C5 2>&1 | tail -2 | cut -c1-700
CFGS="C4 C5 C3 C2" bash scripts/bench_all.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:deposit_lock -s 1 -c 1 \
   -o gpurun_out/${TAG}_lock python bench.py --config C4 --steps 1 --warmup 1 --e2e-steps 0 \
   --no-cpu-baseline > /dev/null 2> gpurun_out/${TAG}_ncu.err; tail -2 gpurun_out/${TAG}_ncu.err
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -15
