# bench (plain) then the ncu launch list of one short bench run
export WN_BENCH_ALLOW_SHORT=1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/benchL.log 2>&1; echo "bench rc=$?"
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plainL.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launchesL.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncuL.log 2>&1; echo "ncu rc=$?"
