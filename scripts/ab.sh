# A/B of library variants: bash scripts/ab.sh base new [more...]
for rep in 1 2; do
  for v in "$@"; do
    WN_LIB_OVERRIDE=$PWD/paper_2510_25159_b200/libwn_$v.so python scripts/build_time.py 2>&1 | tail -1
  done
done
