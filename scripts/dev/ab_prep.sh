# A/B of the per-degree K1 split (PREP_SPLIT) against the single k_prep
bash scripts/ab.sh base sp8 sp16 sp8m
for v in base sp8 sp8m; do
  WN_LIB_OVERRIDE=$PWD/paper_2510_25159_b200/libwn_$v.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_prep|k_deg_bounds" -c 16 --csv python scripts/build_time.py 2>/dev/null | grep -E "k_prep|k_deg" | awk -F'","' -v v=$v '{print v, $5, $NF}' | cut -c1-120
done
WN_LIB_OVERRIDE=$PWD/paper_2510_25159_b200/libwn_sp8.so python -m pytest tests -m gpu -q -x 2>&1 | tail -2
