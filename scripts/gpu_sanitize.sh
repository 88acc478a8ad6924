# compute-sanitizer run of scripts/sanitize_target.py with one tool ($1:
# memcheck | racecheck | synccheck | initcheck), libwn kernels only (namespace
# wn), exact-size allocations (WN_ALLOC_EXACT=1: no caching-allocator slack).
TOOL=${1:-memcheck}
export WN_ALLOC_EXACT=1
EXTRA=""
if [ "$TOOL" = "racecheck" ]; then EXTRA="--racecheck-report all"; fi
if [ "$TOOL" = "memcheck" ]; then EXTRA="--leak-check no --check-api-memory-access yes"; fi
/usr/local/cuda/bin/compute-sanitizer --tool $TOOL $EXTRA --kernel-name kns=_ZN2wn --print-limit 200 \
  --log-file gpurun_out/san_$TOOL.log python scripts/sanitize_target.py > gpurun_out/san_${TOOL}_stdout.log 2>&1
echo "sanitizer $TOOL rc=$?"
tail -5 gpurun_out/san_${TOOL}_stdout.log
tail -5 gpurun_out/san_$TOOL.log
