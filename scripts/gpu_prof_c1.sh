python scripts/prof_step.py --r 32 --iters 60 --kernel-launches 3 > gpurun_out/prof_c1_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python scripts/prof_step.py --r 32 --iters 60 --kernel-launches 3 > gpurun_out/ncu_c1.log 2>&1
for tm in 8 16 32 64; do PDOT_TM=$tm python scripts/prof_step.py --r 32 --iters 60 --kernel-launches 50 2>&1 | tail -1; done
