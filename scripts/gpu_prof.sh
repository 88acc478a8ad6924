export WN_BENCH_ALLOW_SHORT=1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plainp.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_phase1|k_hard" -s 2 -c 2 -o gpurun_out/profp $CMD > gpurun_out/ncup.log 2>&1; echo "ncu rc=$?"
