# occupancy sensitivity of the C4 row kernel: extra dynamic shared memory per CTA lowers the CTAs per SM
# (19.9 KB + 1 KB reserved: 10/SM; +2.9 KB: 9; +5.6 KB: 8; +9.5 KB: 7)
mkdir -p gpurun_out/occ
for x in 0 2900 5600 9500 0; do
  DAXM_ROW_EXTRA_SMEM=$x timeout 300 python bench.py --config C4 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/occ/x$x.json 2> gpurun_out/occ/x$x.err
  python -c "import json; d=json.load(open('gpurun_out/occ/x$x.json')); print('extra smem $x', round(d['ms_per_step'],3), 'ms')" || tail -3 gpurun_out/occ/x$x.err
done
