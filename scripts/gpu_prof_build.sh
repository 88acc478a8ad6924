export WN_BENCH_ALLOW_SHORT=1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plainb.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_prep|k_emit|k_lift" -c 4 -o gpurun_out/profb $CMD > gpurun_out/ncub.log 2>&1; echo "ncu rc=$?"
