# lock-kernel iteration: parity (lock + cutoff tests), C4 variants by build macro, every config, ncu of C4
TAG=${1:-lv}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "lock or cutoff or c1_full or c2_full" 2>&1 | tail -4
CFGS="C4 C5 C3 C2" bash scripts/bench_all.sh
CFG=C4 bash scripts/variants.sh ${VARIANTS:-"dr1:DAXM_LOCK_DR=1" "dr4:DAXM_LOCK_DR=4"}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:deposit_lock -s 1 -c 1 \
   -o gpurun_out/${TAG}_lock python bench.py --config C4 --steps 1 --warmup 1 --e2e-steps 0 \
   --no-cpu-baseline > /dev/null 2> gpurun_out/${TAG}_ncu.err; tail -2 gpurun_out/${TAG}_ncu.err
