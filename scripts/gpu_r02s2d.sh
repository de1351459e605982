# F-staging + plane copy-out: row-path parity, check build, C4/C5 bench vs the previous build (v_base)
T=${TAG:-r02s2d}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "c1_full or c2_full or c2_peaks or c3_full or row_path or zero_skip or both_edges or fused_profile or c5_regions or host_path or graph" > gpurun_out/${T}_pytest.log 2>&1; tail -3 gpurun_out/${T}_pytest.log; grep -E "^E " gpurun_out/${T}_pytest.log | head -8
DAXM_LIBRARY=paper_2201_13309_b200/variants/v_check.so timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "c1_full or c2_full or c3_full or c5_regions" > gpurun_out/${T}_pytest_check.log 2>&1; tail -2 gpurun_out/${T}_pytest_check.log; grep -E "^E " gpurun_out/${T}_pytest_check.log | head -5
ROUNDS=2 CFGS="C4 C5" bash scripts/gpu_libs.sh paper_2201_13309_b200/libdaxm.so paper_2201_13309_b200/variants/v_base.so
timeout 600 python scripts/row_stats.py C4 C5 2>&1 | tail -2 | cut -c1-300
