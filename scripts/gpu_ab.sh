# A/B of library variants under build/ab (one process per config) + GPU tests of the default build
set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf -x > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/gputest.log
for c in ${AB_CFGS:-C5 C2}; do
  AB_CFG=$c timeout 900 python scripts/ab_multi.py build/ab/*.so 2>&1 | tail -12
done
