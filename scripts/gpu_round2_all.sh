# round-2 evidence run: GPU tests, smoke, full bench line, ncu launch list, ncu --set full of the hot kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf -x > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/gputest.log
timeout 300 python __graft_entry__.py 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -c 5000 gpurun_out/bench.log
export WN_BENCH_ALLOW_SHORT=1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-configs"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 || { echo plain failed; tail gpurun_out/plain.log; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncuL.log 2>&1; echo "ncu launches rc=$?"
python scripts/launch_summary.py gpurun_out/launches.csv | cut -c1-120 | head -40
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_phase1|k_hard|k_emit|k_prep|k_lift|k_finish" -s 8 -c 12 -o gpurun_out/prof_full $CMD > gpurun_out/ncuF.log 2>&1; echo "ncu full rc=$?"
ncu -i gpurun_out/prof_full.ncu-rep --page raw --csv > gpurun_out/ncu_full_raw.csv
ncu -i gpurun_out/prof_full.ncu-rep --page details --csv > gpurun_out/ncu_full_details.csv
python scripts/ncu_traffic.py gpurun_out/ncu_full_raw.csv gpurun_out/k_phase1_traffic.json
ncu -i gpurun_out/prof_full.ncu-rep --page source --csv --kernel-name regex:k_phase1 > gpurun_out/p1_source.csv 2>/dev/null
python scripts/ncu_source_hot.py gpurun_out/p1_source.csv 32 0 > gpurun_out/p1_hot.txt
