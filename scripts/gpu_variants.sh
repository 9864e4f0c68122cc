timeout 300 python -m pytest tests/test_gpu_units.py tests/test_gpu_solve.py -x -q 2>&1 | tail -3
for v in s6_b1 s4_b1 s3_b2; do
  PDOT_LIB=paper_2407_19689_b200/lib/libpdot_$v.so timeout 120 python scripts/prof_step.py --iters 30 --kernel-launches 10 2>&1 | tail -1
done
