# usage: bash scripts/gpu_cutoff.sh TAG -- cutoff tests, then C5 pixel-percentage benches with the
# dead-tile zero fill on and off (DAXM_NO_TILE_LIVE), a C4 control, and the launch list of a C5 5 % step.
TAG=${1:-r01}
mkdir -p gpurun_out/cut
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "cutoff or sparse" 2>&1 | tail -3
for f in 0.05 0.5; do
  for v in on off; do
    if [ $v = off ]; then export DAXM_NO_TILE_LIVE=1; else unset DAXM_NO_TILE_LIVE; fi
    timeout 600 python bench.py --config C5 --fraction $f --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
      > gpurun_out/cut/${TAG}_C5_f${f}_${v}.json 2> gpurun_out/cut/${TAG}_C5_f${f}_${v}.err
    python -c "import json; d=json.load(open('gpurun_out/cut/${TAG}_C5_f${f}_${v}.json')); print('C5 f=$f tile_live=$v', round(d['ms_per_step'],3), 'ms active', round(d['config']['active_pixels'],4), 'launches', d['gpu_launches'])" || tail -3 gpurun_out/cut/${TAG}_C5_f${f}_${v}.err
  done
done
unset DAXM_NO_TILE_LIVE
timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/cut/${TAG}_C4.json 2>&1
python -c "import json; d=json.load(open('gpurun_out/cut/${TAG}_C4.json')); print('C4', round(d['ms_per_step'],3), 'ms')"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   -k regex:"deposit|tile_live|zero_dead" --log-file gpurun_out/${TAG}_C5_f0.05_launches.csv \
   python bench.py --config C5 --fraction 0.05 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
tail -12 gpurun_out/${TAG}_C5_f0.05_launches.csv | cut -c1-200
