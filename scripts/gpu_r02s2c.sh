T=${TAG:-r02s2c}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "out_of_core or host_path" > gpurun_out/${T}_pytest.log 2>&1; tail -3 gpurun_out/${T}_pytest.log; grep -E "^E " gpurun_out/${T}_pytest.log | head -8
ROUNDS=2 CFGS="C4 C5" bash scripts/gpu_libs.sh paper_2201_13309_b200/variants/v_base.so paper_2201_13309_b200/variants/v_taug.so
