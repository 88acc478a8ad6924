# Memory / race / init checks without compute-sanitizer (closed on this pool):
#  1. the CHECKED build (device bounds asserts on every derived index, trap on
#     failure) with exact-size, poisoned allocations on the sanitizer target;
#  2. the whole GPU test suite on the CHECKED build with poisoned allocations;
#  3. determinism across launch configurations (default build, poisoned allocations).
set -x
export WN_ALLOC_POISON=1
WN_LIB_OVERRIDE=build/checked/libwn.so WN_ALLOC_EXACT=1 timeout 1200 python scripts/sanitize_target.py > gpurun_out/checked_target.log 2>&1; echo "checked target rc=$?"; tail -16 gpurun_out/checked_target.log
WN_LIB_OVERRIDE=build/checked/libwn.so timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rf > gpurun_out/checked_tests.log 2>&1; echo "checked tests rc=$?"; tail -6 gpurun_out/checked_tests.log
timeout 1200 python scripts/determinism.py > gpurun_out/determinism.log 2>&1; echo "determinism rc=$?"; cat gpurun_out/determinism.log | tail -32
