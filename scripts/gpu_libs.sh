# bench prebuilt library variants (variants/*.so, built here) back to back: usage ROUNDS=2 CFGS="C4" bash scripts/gpu_libs.sh a.so b.so
mkdir -p gpurun_out/libs
for r in $(seq 1 ${ROUNDS:-1}); do
  for c in ${CFGS:-C4}; do
    for lib in "$@"; do
      n=$(basename $lib .so)
      DAXM_LIBRARY=$lib timeout 300 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline ${EXTRA} > gpurun_out/libs/${n}_${c}.json 2> gpurun_out/libs/${n}_${c}.err
      python -c "import json; d=json.load(open('gpurun_out/libs/${n}_${c}.json')); print('round $r', '$c', '$n', round(d['ms_per_step'],3), 'ms frac', round(d['roofline']['frac'],3), 'parity', (d.get('parity_sample') or {}).get('pass'))" || tail -3 gpurun_out/libs/${n}_${c}.err
    done
  done
done
