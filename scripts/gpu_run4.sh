python scripts/dbg_c3.py 2>&1 | tail -30
python -m pytest tests -m gpu -q 2>&1 | tail -15
