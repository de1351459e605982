# new GPU tests (NaN corner pairs, out-of-core host ring) + row admission stats + variant A/B on C4
T=${TAG:-r02s2b}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "nan_corner or out_of_core or host_path" > gpurun_out/${T}_pytest.log 2>&1; tail -3 gpurun_out/${T}_pytest.log; grep -E "^E " gpurun_out/${T}_pytest.log | head -8
timeout 300 python scripts/row_stats.py C4 C5 2>&1 | tail -2 | cut -c1-400
ROUNDS=2 CFGS="C4" bash scripts/gpu_libs.sh paper_2201_13309_b200/variants/v_base.so paper_2201_13309_b200/variants/v_pb8.so paper_2201_13309_b200/variants/v_nb16.so paper_2201_13309_b200/variants/v_lb14.so paper_2201_13309_b200/variants/v_nb16lb14.so
for n in nb16 lb14; do python -c "import json; d=json.load(open('gpurun_out/libs/v_${n}_C4.json')); print('$n', d['plan'])"; done
