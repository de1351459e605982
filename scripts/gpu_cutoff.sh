# usage: bash scripts/gpu_cutoff.sh TAG -- cutoff tests, then C5 pixel-percentage benches: the dead-tile
# zero fill off (DAXM_NO_TILE_LIVE) and on with DAXM_ZERO_PER_SM fill blocks per SM, a C4 control, and
# the launch list of a C5 5 % step.
TAG=${1:-r01}
PER_SM=${PER_SM:-"1 2 4 8"}
mkdir -p gpurun_out/cut
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "cutoff or sparse" 2>&1 | tail -3
run() {  # run NAME FRACTION [env...]
  local name=$1 f=$2; shift 2
  env "$@" timeout 600 python bench.py --config C5 --fraction $f --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
    > gpurun_out/cut/${TAG}_${name}.json 2> gpurun_out/cut/${TAG}_${name}.err
  python -c "import json; d=json.load(open('gpurun_out/cut/${TAG}_${name}.json')); print('${name}', round(d['ms_per_step'],3), 'ms active', round(d['config']['active_pixels'],4), 'launches', d['gpu_launches'])" || tail -3 gpurun_out/cut/${TAG}_${name}.err
}
run C5_f0.05_off 0.05 DAXM_NO_TILE_LIVE=1
run C5_f0.05_tile 0.05 DAXM_NO_GRP_LIVE=1
for n in $PER_SM; do run C5_f0.05_z$n 0.05 DAXM_ZERO_PER_SM=$n; done
run C5_f0.5_tile 0.5 DAXM_NO_GRP_LIVE=1
run C5_f0.5 0.5
run C5_f0.25 0.25
timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/cut/${TAG}_C4.json 2>&1
python -c "import json; d=json.load(open('gpurun_out/cut/${TAG}_C4.json')); print('C4', round(d['ms_per_step'],3), 'ms')"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   -k regex:"deposit|tile_live|zero_dead" --log-file gpurun_out/${TAG}_C5_f0.05_launches.csv \
   python bench.py --config C5 --fraction 0.05 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
grep -c zero_dead gpurun_out/${TAG}_C5_f0.05_launches.csv
