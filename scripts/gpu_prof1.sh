set -x
python scripts/prof_step.py --iters 30 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v1.csv python scripts/prof_step.py --iters 30 > gpurun_out/ncu_launch.log 2>&1
python scripts/prof_step.py --iters 5 > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 8 -c 1 -o gpurun_out/prof_step_v1 python scripts/prof_step.py --iters 5 > gpurun_out/ncu_full.log 2>&1
echo done
