# gpu_ab.sh plus the DAXM_ROW_CHECK build's parity (schedule violations counted in the kernel)
T=${TAG:-r02ab}
DAXM_LIBRARY=paper_2201_13309_b200/variants/v_check.so timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "c1_full or c2_full or c3_full or c5_regions" > gpurun_out/${T}_pytest_check.log 2>&1; tail -1 gpurun_out/${T}_pytest_check.log; grep -E "^E " gpurun_out/${T}_pytest_check.log | head -5
bash scripts/gpu_ab.sh "$@"
