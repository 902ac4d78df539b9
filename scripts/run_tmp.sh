timeout 600 python scripts/prof_c3.py 28 c4 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
