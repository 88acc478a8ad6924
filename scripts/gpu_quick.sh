python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python scripts/devtime.py C2 C4 2>&1 | grep -E "^C" | cut -c1-150
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/benchq.log 2>&1; grep -o '"ms_per_step": [0-9.]*\|"query_only": {"ms": [0-9.]*\|"k3_ms": [0-9.]*' gpurun_out/benchq.log
