# screened STEP pass: bit-identity tests, full GPU suite, C3/C1 bench
set -x
timeout 900 python -m pytest tests/test_gpu_screen.py -x -q -s 2>&1 | tail -30
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 600 python bench.py --no-cpu > gpurun_out/scr_c3.json 2> gpurun_out/scr_c3.err; echo c3 rc=$?
tail -5 gpurun_out/scr_c3.err
PDOT_SCREEN=0 timeout 600 python bench.py --no-cpu --no-variant --no-e2e > gpurun_out/dense_c3.json 2> gpurun_out/dense_c3.err; echo dense rc=$?
timeout 600 python bench.py --config c1 --no-cpu > gpurun_out/scr_c1.json 2> gpurun_out/scr_c1.err; echo c1 rc=$?
