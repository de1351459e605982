python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CFG=C4 bash scripts/variants.sh "old:DAXM_SHPROD=0,DAXM_LASTSTORE=0" "shprod:DAXM_LASTSTORE=0" "last:DAXM_SHPROD=0" "both:" "old2:DAXM_SHPROD=0,DAXM_LASTSTORE=0" "both2:"
CFG=C5 bash scripts/variants.sh "c5old:DAXM_SHPROD=0,DAXM_LASTSTORE=0" "c5both:"
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x 2>&1 | tail -3
