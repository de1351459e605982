# quick perf iteration: bench (no e2e/cpu) + ncu capture of the fast kernel
TAG=${1:-q}; CFG=${2:-C4}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python bench.py --config $CFG --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; tail -3 gpurun_out/${TAG}_bench.err; python -c "
import json; d=json.load(open('gpurun_out/${TAG}_bench.json')); print('ms', d['ms_per_step'], 'GB/s', d['roofline']['achieved'], 'frac', d['roofline']['frac'], d['plan'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:deposit_fast -s 1 -c 1 \
   -o gpurun_out/${TAG}_deposit python bench.py --config $CFG --steps 1 --warmup 1 --e2e-steps 0 \
   --no-cpu-baseline > /dev/null 2> gpurun_out/${TAG}_ncu.err; tail -2 gpurun_out/${TAG}_ncu.err
