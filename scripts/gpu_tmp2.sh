timeout 300 python scripts/k2_trace.py 128 400 2>&1 | tail -5
