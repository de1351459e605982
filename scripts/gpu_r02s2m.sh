T=${TAG:-r02s2m}
for L in paper_2201_13309_b200/libdaxm.so paper_2201_13309_b200/variants/v_m4.so; do DAXM_LIBRARY=$L timeout 300 python scripts/row_stats.py C4 C5 2>&1 | tail -2 | cut -c1-330; done
NONCU=1 ROUNDS=2 TAG=$T bash scripts/gpu_ab_check.sh "$@"
