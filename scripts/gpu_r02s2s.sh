T=${TAG:-r02s2s}
timeout 300 python scripts/row_stats.py C4 C4:trailing 2>&1 | tail -2 | cut -c1-330
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/${T}_C4_launches.csv python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/${T}_C4t_launches.csv python bench.py --edge trailing --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/ | tail -3
