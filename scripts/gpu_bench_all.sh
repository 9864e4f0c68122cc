python bench.py --config c3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3 rc=$?
python bench.py --config c1 --no-cpu > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo c1 rc=$?
python bench.py --config c2 --no-cpu > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2 rc=$?
python bench.py --config c4 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4 rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
