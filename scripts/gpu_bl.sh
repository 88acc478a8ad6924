# ncu launch lists of the build kernels for library variants given as paths: bash scripts/gpu_bl.sh build/ab/x.so ...
for v in "$@"; do
  b=$(basename $v .so)
  WN_LIB_OVERRIDE=$PWD/$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_prep|k_emit|k_lift|k_s0pre|k_plan|k_deg|k_loop|k_csr|k_iota|Radix|Scan" -c 120 --csv --log-file gpurun_out/bl_$b.csv python scripts/build_time.py > /dev/null 2>&1
  echo "== $b"; python scripts/launch_summary.py gpurun_out/bl_$b.csv | cut -c1-110 | head -24
done
