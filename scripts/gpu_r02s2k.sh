T=${TAG:-r02s2k}
timeout 300 python scripts/row_stats.py C2 C3 C4 C5 C2:trailing 2>&1 | tail -5 | cut -c1-250
TAG=$T bash scripts/gpu_ab_check.sh "$@"
