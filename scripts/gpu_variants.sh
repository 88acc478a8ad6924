python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for lib in "" scripts/dev/libwn_q1.so scripts/dev/libwn_q4.so; do
  echo "== lib=$lib"
  WN_LIB_OVERRIDE=$lib python scripts/devtime.py C2 C3 2>&1 | grep -E "^C" | cut -c1-110
  WN_LIB_OVERRIDE=$lib python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bv.log 2>&1; grep -o '"ms_per_step": [0-9.]*\|"query_only": {"ms": [0-9.]*\|"k3_ms": [0-9.]*' gpurun_out/bv.log
done
