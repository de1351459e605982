python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CFG=C4 bash scripts/variants.sh "base:" "advA:DAXM_ADV=1" "advAB:DAXM_ADV=1,DAXM_NOCLAMP=1" "advABC:DAXM_ADV=1,DAXM_NOCLAMP=1,DAXM_RCP1=1" "base2:"
CFG=C5 bash scripts/variants.sh "c5base:" "c5advA:DAXM_ADV=1"
