CMD="python bench.py --steps 40 --warmup 5 --no-e2e --no-cpu --no-tol --no-variant"
$CMD > gpurun_out/ncu_bench_plain.json 2> gpurun_out/ncu_bench_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_v3.csv $CMD > gpurun_out/ncu_bench.log 2>&1
echo launch-list rc=$?
python scripts/prof_step.py --iters 5 --kernel-launches 1 > gpurun_out/prof_v3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:stream_kernel -s 1 -c 1 -o gpurun_out/prof_step_v3 python scripts/prof_step.py --iters 5 --kernel-launches 1 > gpurun_out/ncu_v3.log 2>&1
echo full rc=$?
