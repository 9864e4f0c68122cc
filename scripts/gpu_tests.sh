set -x
nvidia-smi --query-gpu=name --format=csv
python -c "import __graft_entry__" 2>/dev/null
timeout 600 python -m pytest tests/test_gpu_units.py -x -q 2>&1 | tail -30
timeout 900 python -m pytest tests/test_gpu_solve.py -x -q -s 2>&1 | tail -40
