nvidia-smi --query-gpu=memory.total,memory.used --format=csv
timeout 1200 python scripts/big_check.py 181 120 2>&1 | tail -4
