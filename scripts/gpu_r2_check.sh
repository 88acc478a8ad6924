# round-2 GPU check: full GPU test suite, smoke, full-size parity report
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; }
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -40 gpurun_out/gputest.log
timeout 300 python __graft_entry__.py 2>&1 | tail -3
timeout 1500 python scripts/parity_full.py --out gpurun_out/PARITY_r02.json > gpurun_out/parity.log 2>&1; echo "parity rc=$?"; cut -c1-400 gpurun_out/parity.log
