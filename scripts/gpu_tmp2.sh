timeout 1800 python -m pytest -q -x tests -m gpu 2>&1 | tail -2
timeout 600 python bench.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['traffic'], d['screening']['k1_us'], d['e2e']['value'], d['time_to_tol']['seconds'])"
