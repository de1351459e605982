# C4 bench under environment-variable experiment knobs: "NAME:VAR=VAL,VAR=VAL" ...
mkdir -p gpurun_out/envvar
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for spec in "$@"; do
  name=${spec%%:*}; envs=${spec#*:}
  env $(echo $envs | tr ',' ' ') timeout 300 python bench.py --config ${CFG:-C4} --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/envvar/${name}.json 2> gpurun_out/envvar/${name}.err
  python -c "import json; d=json.load(open('gpurun_out/envvar/${name}.json')); print('${name}', '${envs}', round(d['ms_per_step'],3), 'ms', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/envvar/${name}.err
done
