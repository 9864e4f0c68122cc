python scripts/prof_step.py --r 128 --iters 12 --kernel-launches 1 > gpurun_out/pf_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:finalize -s 8 -c 1 -o gpurun_out/prof_fin_c3 python scripts/prof_step.py --r 128 --iters 12 --kernel-launches 1 > gpurun_out/ncu_fin3.log 2>&1
python scripts/prof_step.py --r 32 --iters 12 --kernel-launches 1 > gpurun_out/pf_plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:finalize -s 8 -c 1 -o gpurun_out/prof_fin_c1 python scripts/prof_step.py --r 32 --iters 12 --kernel-launches 1 > gpurun_out/ncu_fin1.log 2>&1
echo rc=$?
