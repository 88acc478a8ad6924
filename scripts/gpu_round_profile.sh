# Full bench line + launch list + ncu --set full of the hot kernels (C5 step)
set -x
python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
export WN_BENCH_ALLOW_SHORT=1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 || { echo plain failed; tail gpurun_out/plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncuL.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_phase1|k_hard|k_emit|k_prep|k_lift" -s 5 -c 5 -o gpurun_out/prof_full $CMD > gpurun_out/ncuF.log 2>&1; echo "ncu full rc=$?"
python scripts/ncu_k3_metrics.py gpurun_out/prof_full.ncu-rep gpurun_out/plain.log gpurun_out/k_phase1_metrics.json
ncu -i gpurun_out/prof_full.ncu-rep --page raw --csv > gpurun_out/ncu_full_raw.csv
ncu -i gpurun_out/prof_full.ncu-rep --page details --csv > gpurun_out/ncu_full_details.csv
python scripts/launch_summary.py gpurun_out/launches.csv | cut -c1-110 | head -20
