# parity of the default build (smoke + lock/cutoff tests), then prebuilt variants back to back
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "lock or cutoff or c1_full or c2_full" 2>&1 | tail -3
ROUNDS=${ROUNDS:-1} CFGS="${CFGS:-C4 C3}" bash scripts/gpu_libs.sh "$@"
