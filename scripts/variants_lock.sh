# build lock-kernel variants (in-tree, travel with gpurun), then bench each on C4
set -e
mkdir -p variants
python - <<'PY'
from paper_2201_13309_b200 import _build
V = {"u1m4": ["DAXM_LOCK_UNROLL=1", "DAXM_LOCK_MINB=4"], "u2m3": ["DAXM_LOCK_UNROLL=2", "DAXM_LOCK_MINB=3"],
     "u1m3": ["DAXM_LOCK_UNROLL=1", "DAXM_LOCK_MINB=3"], "u2m4": ["DAXM_LOCK_UNROLL=2", "DAXM_LOCK_MINB=4"]}
for k, d in V.items():
    _build.build_library(out=f"variants/{k}.so", defines=d)
PY
