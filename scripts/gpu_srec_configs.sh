# slack certificates on / off (PDOT_SREC=0) on C2 and C4: complete-solve bench lines, alternating, twice
set -x
mkdir -p gpurun_out
for rep in 1 2; do
  for c in c2 c4; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-variant > gpurun_out/src_on_${c}_$rep.json 2>/dev/null
    PDOT_SREC=0 timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-variant > gpurun_out/src_off_${c}_$rep.json 2>/dev/null
  done
done
