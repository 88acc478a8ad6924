set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q -x 2>&1 | tail -15
python __graft_entry__.py 2>&1 | tail -3
python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"; tail -c 4000 gpurun_out/bench_full.log
