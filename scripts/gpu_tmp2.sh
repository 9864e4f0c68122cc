timeout 1800 python -m pytest -q -x tests -m gpu 2>&1 | tail -3
