python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"; tail -c 4000 gpurun_out/bench_full.log
export WN_BENCH_ALLOW_SHORT=1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plainL.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncuL.log 2>&1; echo "ncu launches rc=$?"
$CMD > gpurun_out/plainF.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_phase1|k_hard|k_finish|k_overflow" -s 4 -c 4 -o gpurun_out/prof_full $CMD > gpurun_out/ncuF.log 2>&1; echo "ncu full rc=$?"
