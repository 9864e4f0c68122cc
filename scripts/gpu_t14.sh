timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --config c1 --no-cpu --no-e2e > gpurun_out/b_c1.json 2>&1; python bench.py --config c3 --no-cpu --no-e2e > gpurun_out/b_c3.json 2>&1
python scripts/prof_step.py --r 32 --iters 60 --kernel-launches 3 > gpurun_out/pc1.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1b.csv python scripts/prof_step.py --r 32 --iters 60 --kernel-launches 3 > /dev/null 2>&1
python scripts/prof_step.py --r 128 --iters 30 --kernel-launches 3 > gpurun_out/pc3.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3b.csv python scripts/prof_step.py --r 128 --iters 30 --kernel-launches 3 > /dev/null 2>&1
