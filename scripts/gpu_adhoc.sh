python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CFG=C4 bash scripts/variants.sh "h2000:" "h0:DAXM_HINT=0" "h100:DAXM_HINT=100" "h500:DAXM_HINT=500" "h10000:DAXM_HINT=10000" "h2000b:" 2>&1 | grep -v warning
