# developer loop: GPU tests, a short bench line, host-phase trace of one build, launch list
set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf -x > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/gputest.log
export WN_BENCH_ALLOW_SHORT=1
timeout 900 python bench.py --steps 10 --no-e2e --no-cpu-baseline --no-configs > gpurun_out/bench_dev.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/bench_dev.log"):
    if l.startswith("{"):
        d = json.loads(l)
        r = d["roofline"]
        print("step %.3f ms  query %.3f ms  p1 %.3f  k3 %.3f  frac %.3f  grid step %.3f query %.3f" % (
            d["ms_per_step"], d["query_only"]["ms"], r["kernel_ms"], r["k3"]["ms"], r["frac"], d["grid"]["ms_per_step"], d["grid"]["query_ms"]))
        print(d["counters"])
PY
timeout 300 python scripts/trace_build.py 2>&1 | tail -12
TRACE_MODE=2 timeout 300 python scripts/trace_build.py 2>&1 | tail -12
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-configs"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncuL.log 2>&1; echo "ncu launches rc=$?"
python scripts/launch_summary.py gpurun_out/launches.csv | cut -c1-100 | head -24
