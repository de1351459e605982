# usage: bash scripts/gpu_record.sh TAG -- the measurement pass for the record:
# default bench line, every config, C5 pixel percentages, launch list + ncu full of C4.
TAG=${1:-r01}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err
cat gpurun_out/${TAG}_bench_default.json; tail -2 gpurun_out/${TAG}_bench_default.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2>&1
cat gpurun_out/${TAG}_bench_reference.json | tail -1
CFGS="C2 C3 C4 C5" bash scripts/bench_all.sh
for f in 0.5 0.25 0.05; do
  timeout 600 python bench.py --config C5 --fraction $f --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/all/C5_f$f.json 2> gpurun_out/all/C5_f$f.err
  python -c "import json; d=json.load(open('gpurun_out/all/C5_f$f.json')); print('C5 fraction $f', round(d['ms_per_step'],3), 'ms active', round(d['config']['active_pixels'],4))" || tail -3 gpurun_out/all/C5_f$f.err
done
bash scripts/gpu_profile.sh ${TAG} C4
