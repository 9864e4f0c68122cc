timeout 900 python -m pytest -q -x tests/test_gpu_screen.py 2>&1 | tail -2
timeout 300 python scripts/k2_trace.py 128 400 2>&1 | grep -E "timeline"
timeout 300 python scripts/k2_trace.py 128 1000 2>&1 | grep -E "timeline"
timeout 600 python bench.py --config c3 --no-cpu --no-e2e --no-variant 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['screening']['k1_us'], d['time_to_tol']['seconds'], d['time_to_tol']['iterations'])"
