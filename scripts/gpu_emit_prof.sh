for v in "$@"; do
  WN_LIB_OVERRIDE=$PWD/paper_2510_25159_b200/libwn_$v.so ncu --set full --clock-control none --import-source on -k regex:"k_emit|k_cold" -s 4 -c 2 -o gpurun_out/emit_$v python scripts/build_time.py > /dev/null 2>&1
  ncu -i gpurun_out/emit_$v.ncu-rep --page raw --csv > gpurun_out/emit_$v.csv 2>/dev/null
done
