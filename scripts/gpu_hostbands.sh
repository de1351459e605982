# in-core host pipeline: 16 vs 8 row bands (e2e of the default C4 bench line), host-path tests
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "host_path" 2>&1 | tail -1
for L in paper_2201_13309_b200/libdaxm.so paper_2201_13309_b200/variants/v_hb16.so; do
  DAXM_LIBRARY=$L timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 5 --no-cpu-baseline > gpurun_out/hb_$(basename $L .so).json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/hb_$(basename $L .so).json')); e=d['e2e']; print('$L e2e', round(e['ms_per_step'],1), 'ms pcie frac', round(e['pcie_roofline']['frac'],3))"
done
