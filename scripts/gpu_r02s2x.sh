for L in paper_2201_13309_b200/libdaxm.so paper_2201_13309_b200/variants/v_rmw.so; do
  DAXM_LIBRARY=$L timeout 600 python bench.py --config C4 --edge both --steps 5 --warmup 2 --e2e-steps 0 --no-cpu-baseline > gpurun_out/both_$(basename $L .so).json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/both_$(basename $L .so).json')); print('$L C4 both', round(d['ms_per_step'],3), d.get('parity_sample'))"
done
DAXM_LIBRARY=paper_2201_13309_b200/variants/v_rmw.so timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "both" 2>&1 | tail -2
