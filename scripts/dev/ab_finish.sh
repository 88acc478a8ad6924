# A/B of the k_finish load unroll (FINISH_UNROLL 1 / 4 / 8)
bash scripts/ab.sh base f4 f8
for v in base f4 f8; do
  WN_LIB_OVERRIDE=$PWD/paper_2510_25159_b200/libwn_$v.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_finish -c 3 --csv python scripts/build_time.py 2>/dev/null | grep k_finish | awk -F'","' -v v=$v '{print v, $NF}'
done
WN_LIB_OVERRIDE=$PWD/paper_2510_25159_b200/libwn_f4.so python -m pytest tests -m gpu -q -x 2>&1 | tail -2
