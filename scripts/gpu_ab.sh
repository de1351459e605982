# quick A/B of the current library: row-path parity subset, C4/C5 bench against variants/v_base.so,
# one ncu --set full capture of the C4 row kernel.  usage: TAG=... bash scripts/gpu_ab.sh [extra libs]
T=${TAG:-r02ab}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "c1_full or c2_full or c3_full or row_path or zero_skip or both_edges_mode or fused_profile or c5_regions" > gpurun_out/${T}_pytest.log 2>&1; tail -2 gpurun_out/${T}_pytest.log; grep -E "^E " gpurun_out/${T}_pytest.log | head -6
ROUNDS=${ROUNDS:-1} CFGS="${CFGS:-C4 C5}" bash scripts/gpu_libs.sh paper_2201_13309_b200/libdaxm.so paper_2201_13309_b200/variants/v_base.so "$@"
[ -n "$NONCU" ] || TAG=${T} bash scripts/gpu_ncu_var.sh
