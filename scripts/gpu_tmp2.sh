timeout 900 python -m pytest -q -x tests/test_gpu_screen.py tests/test_gpu_shard.py 2>&1 | tail -2
timeout 600 python bench.py --config c3 --no-cpu --no-e2e --no-variant 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['time_to_tol'])"
