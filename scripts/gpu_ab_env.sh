# A/B of an env-gated variant: $1 = VAR=value; runs the screening parity tests
# under the variant, then C3 / C2 bench lines for both arms and a pass timeline
set -x
V="$1"
env $V timeout 900 python -m pytest tests/test_gpu_screen.py tests/test_gpu_solve.py -x -q 2>&1 | tail -4
for c in c3 c2; do
  timeout 600 python bench.py --config $c --no-cpu --no-variant > gpurun_out/ab_base_$c.json 2> gpurun_out/ab_base_$c.err; echo base $c rc=$?
  env $V timeout 600 python bench.py --config $c --no-cpu --no-variant > gpurun_out/ab_var_$c.json 2> gpurun_out/ab_var_$c.err; echo var $c rc=$?
done
env $V timeout 300 python scripts/k2_trace.py 128 400 > gpurun_out/ab_var_trace.txt 2>&1; echo trace rc=$?
