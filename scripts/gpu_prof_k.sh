# ncu --set full of the kernels matching $1 (regex), first $2 launches, of one short bench run
export WN_BENCH_ALLOW_SHORT=1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plaink.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"$1" -c ${2:-1} -o gpurun_out/profk $CMD > gpurun_out/ncuk.log 2>&1; echo "ncu rc=$?"
