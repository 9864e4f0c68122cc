# --set full captures (source, dense warp sampling) of the screened-pass kernels
# in mid-solve of a 500-iteration C3 solve; run after the plain driver exits 0
set -x
mkdir -p gpurun_out
P="python scripts/prof_solve.py 128 500"
$P > gpurun_out/prof_solve.json 2>&1; echo prof_solve rc=$?
for k in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:$k \
    --launch-skip 300 --launch-count 1 -o gpurun_out/k1p_$k -f $P > /dev/null 2>gpurun_out/ncu_$k.err; echo $k rc=$?
done
