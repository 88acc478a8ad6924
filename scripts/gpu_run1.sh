set -x
python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench1.log
export WN_BENCH_ALLOW_SHORT=1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_query -s 1 -c 1 -o gpurun_out/prof_k3 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
tail -5 gpurun_out/ncu_full.log
