python -m pytest tests -m gpu -x -q 2>&1 | tail -15
WN_TRACE=1 python scripts/devtime.py C1 C2 C3 C4 2>&1 | grep -v "^\[wn_build\]" | tail -12
WN_TRACE=1 python scripts/devtime.py C5 2>&1 | tail -30
