set -x
python bench.py --steps 300 --warmup 20 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo rc=$?
cat gpurun_out/bench_c3.json; tail -5 gpurun_out/bench_c3.err
