timeout 600 python bench.py --no-cpu > gpurun_out/scr_c3.json 2> gpurun_out/scr_c3.err; echo c3 rc=$?
timeout 600 python bench.py --config c1 --no-cpu > gpurun_out/scr_c1.json 2> gpurun_out/scr_c1.err; echo c1 rc=$?
PDOT_SCREEN=1 timeout 600 python bench.py --config c1 --no-cpu --no-e2e --no-variant > gpurun_out/scr_c1s.json 2> gpurun_out/scr_c1s.err; echo c1s rc=$?
timeout 600 python bench.py --config c2 --no-cpu > gpurun_out/scr_c2.json 2> gpurun_out/scr_c2.err; echo c2 rc=$?
PDOT_SCREEN=0 timeout 600 python bench.py --config c2 --no-cpu --no-e2e --no-variant > gpurun_out/scr_c2d.json 2> gpurun_out/scr_c2d.err; echo c2d rc=$?
