# ncu launch list of one bench step (C5) + per-kernel summary
export WN_BENCH_ALLOW_SHORT=1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 || { echo plain failed; tail gpurun_out/plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncuL.log 2>&1; echo "ncu launches rc=$?"
python scripts/launch_summary.py gpurun_out/launches.csv | cut -c1-110 | head -24
