timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/scr_c3.json 2> gpurun_out/scr_c3.err; echo c3 rc=$?
