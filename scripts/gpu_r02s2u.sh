# lock-check build test (merged step-locked template), old-path tests, and the DRAM traffic of one
# C4 / C5 step (sum over the class launches) for bench.py's roofline.traffic
T=${TAG:-r02s2u}
mkdir -p gpurun_out/$T
timeout 1500 python -m pytest tests/test_parity_gpu.py -x -q -k "lock or overlap or fast_kernel or general_kernel or cutoff_dead or graph" > gpurun_out/$T/pytest.log 2>&1; tail -2 gpurun_out/$T/pytest.log; grep -E "^E " gpurun_out/$T/pytest.log | head -5
for c in C4 C5; do
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$T/${c}_dram.csv python bench.py --config $c --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
done
ls gpurun_out/$T
