# QPL A/B + GPU tests of the QPL=2 variant (the test suite on the variant through WN_LIB_OVERRIDE)
set -x
WN_LIB_OVERRIDE=build/ab/libwn_a_k1s.so timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rf -x > gpurun_out/gputest_ab.log 2>&1; echo "pytest ab rc=$?"; tail -8 gpurun_out/gputest_ab.log
for c in C5 C2 C3; do
  AB_CFG=$c timeout 900 python scripts/ab_multi.py build/ab/*.so 2>&1 | tail -4
done
