# per-launch kernel times (ncu, cold, serialised) of a short bench run: usage TAG CFG [extra bench args]
TAG=${1:-l}; CFG=${2:-C4}; shift 2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv -k regex:"deposit" \
   --log-file gpurun_out/${TAG}_launches.csv python bench.py --config $CFG --steps 1 --warmup 1 --e2e-steps 0 \
   --no-cpu-baseline "$@" > /dev/null 2> gpurun_out/${TAG}_launches.err
python - gpurun_out/${TAG}_launches.csv <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; d = collections.defaultdict(dict)
for r in rows[1:]:
    x = dict(zip(h, r)); d[(x['ID'], x['Kernel Name'][:60], x['Grid Size'])][x['Metric Name']] = x['Metric Value']
for k, v in d.items(): print(k, v)
PY
