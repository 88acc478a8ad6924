python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python scripts/devtime.py C2 C3 C4 2>&1 | tail -8
WN_TRACE=1 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench3.log 2>&1; tail -c 2500 gpurun_out/bench3.log
export WN_BENCH_ALLOW_SHORT=1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_phase1|k_hard" -s 2 -c 2 -o gpurun_out/prof3 $CMD > gpurun_out/ncu3.log 2>&1; echo "ncu rc=$?"
