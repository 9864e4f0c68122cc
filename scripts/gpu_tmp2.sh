timeout 900 python -m pytest -q tests/test_gpu_screen.py 2>&1 | tail -2
