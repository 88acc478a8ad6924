bash scripts/ab.sh base s64 w1 w2
for v in base s64 w1 w2; do
  WN_LIB_OVERRIDE=$PWD/paper_2510_25159_b200/libwn_$v.so ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_emit -c 4 --csv python scripts/build_time.py 2>/dev/null | grep k_emit | awk -F'","' -v v=$v '{print v, $(NF-2), $NF}'
done
