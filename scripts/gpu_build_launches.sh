# ncu launch lists of the build kernels for library variants: bash scripts/gpu_build_launches.sh v1 v2
for v in "$@"; do
  WN_LIB_OVERRIDE=$PWD/paper_2510_25159_b200/libwn_$v.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_prep|k_emit|k_cold|k_cold_slots|k_lift|k_s0pre|k_plan|k_deg|k_loop" -c 40 --csv --log-file gpurun_out/bl_$v.csv python scripts/build_time.py > /dev/null 2>&1
  echo "== $v"; python scripts/launch_summary.py gpurun_out/bl_$v.csv | cut -c1-100
done
