# GPU tests + bench line + ncu launch list of one C5 step
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; }
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf -x > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/gputest.log
timeout 300 python __graft_entry__.py 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -c 6000 gpurun_out/bench.log
export WN_BENCH_ALLOW_SHORT=1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-configs"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncuL.log 2>&1; echo "ncu launches rc=$?"
python scripts/launch_summary.py gpurun_out/launches.csv | cut -c1-120 | head -40
