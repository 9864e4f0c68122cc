python scripts/prof_step.py --iters 30 --kernel-launches 3 > gpurun_out/prof3_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v2.csv python scripts/prof_step.py --iters 30 --kernel-launches 3 > gpurun_out/ncu3_launch.log 2>&1
python scripts/prof_step.py --iters 5 --kernel-launches 1 > gpurun_out/prof3_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:stream_kernel -s 1 -c 1 -o gpurun_out/prof_step_v2 python scripts/prof_step.py --iters 5 --kernel-launches 1 > gpurun_out/ncu3_full.log 2>&1
echo rc=$?
