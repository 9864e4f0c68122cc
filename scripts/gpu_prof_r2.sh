# Round-2 ncu evidence for the screened pass at C3 (run each only after the plain
# command exits 0): the launch list of a short bench run, and one --set full
# capture (with source) of K0 screen_kernel, K1 unit_kernel, K1b tile_kernel and
# K2 finalize_kernel in mid-solve of a 500-iteration C3 solve.
set -x
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-variant --no-cpu"
$B > gpurun_out/prof_plain.json 2>gpurun_out/prof_plain.err; echo plain rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_r2.csv $B > /dev/null 2>gpurun_out/ncu_l.err; echo launches rc=$?
P="python scripts/prof_solve.py 128 500"
$P > gpurun_out/prof_solve.json 2>&1; echo prof_solve rc=$?
for k in unit_kernel screen_kernel tile_kernel finalize_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 300 --launch-count 1 -o gpurun_out/full_r2_$k -f $P > /dev/null 2>gpurun_out/ncu_$k.err; echo $k rc=$?
done
