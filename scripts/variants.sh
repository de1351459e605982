# Build kernel variants (-D flags) and bench each (device-resident, no e2e/cpu baseline).
# usage: CFG=C4 bash scripts/variants.sh "NAME1:DEF1,DEF2" "NAME2:DEF" ...
mkdir -p gpurun_out/variants
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  python - "$name" "$defs" <<'PY'
import sys
from paper_2201_13309_b200 import _build
name, defs = sys.argv[1], sys.argv[2]
d = [x for x in defs.split(",") if x]
_build.build_library(force=True, out=f"gpurun_out/variants/lib_{name}.so", defines=d)
PY
  DAXM_LIBRARY=gpurun_out/variants/lib_${name}.so timeout 300 python bench.py --config ${CFG:-C4} --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/variants/${name}.json 2> gpurun_out/variants/${name}.err
  python -c "import json,sys; d=json.load(open('gpurun_out/variants/${name}.json')); print('${name}', '${defs}', round(d['ms_per_step'],3), 'ms', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/variants/${name}.err
done
