timeout 900 python -m pytest tests/test_gpu_screen.py -x -q 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 600 python bench.py --no-cpu --no-e2e --no-variant > gpurun_out/scr_c3.json 2> gpurun_out/scr_c3.err; echo c3 rc=$?
timeout 300 python scripts/k2_trace.py 128 400 2>&1 | tail -1
B="python bench.py --steps 120 --warmup 5 --no-tol --no-e2e --no-variant --no-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 2000 --csv --log-file gpurun_out/launches_unit_warm.csv $B > /dev/null 2>gpurun_out/ncu2.err; echo ncu2 rc=$?
