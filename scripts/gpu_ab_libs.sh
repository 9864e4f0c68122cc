# A/B of prebuilt library variants: each argument names lib/variants/<name>.so;
# C3 and C2 bench lines per variant plus a pass timeline
set -x
for v in "$@"; do
  L=paper_2407_19689_b200/lib/variants/$v.so
  PDOT_LIB=$L timeout 600 python -m pytest tests/test_gpu_screen.py -x -q 2>&1 | tail -2
  for c in c3 c2; do
    PDOT_LIB=$L timeout 600 python bench.py --config $c --no-cpu --no-variant > gpurun_out/ab_${v}_$c.json 2> gpurun_out/ab_${v}_$c.err; echo $v $c rc=$?
  done
  PDOT_LIB=$L timeout 300 python scripts/k2_trace.py 128 400 > gpurun_out/ab_${v}_trace.txt 2>&1
done
