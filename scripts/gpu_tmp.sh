timeout 900 python -m pytest tests/test_gpu_screen.py -x -q 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python scripts/k2_trace.py 128 400 2>&1 | grep -E "timeline|per pass"
timeout 600 python bench.py --no-cpu --no-e2e --no-variant > gpurun_out/scr_c3.json 2> gpurun_out/scr_c3.err; echo c3 rc=$?
