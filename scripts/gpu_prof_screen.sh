# ncu evidence for the screened pass at C3: launch list of a short bench run and one
# --set full capture each of the K0 / K1 / K2 kernels in mid-solve.
set -x
B="python bench.py --steps 60 --warmup 5 --no-tol --no-e2e --no-variant --no-cpu"
$B > gpurun_out/prof_plain.json 2>/dev/null; echo plain rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_screen.csv $B > /dev/null 2>gpurun_out/ncu1.err; echo ncu1 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 1200 --csv --log-file gpurun_out/launches_screen_warm.csv $B > /dev/null 2>gpurun_out/ncu2.err; echo ncu2 rc=$?
for k in sparse_kernel screen_kernel finalize_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 80 --launch-count 1 -o gpurun_out/full_$k -f $B > /dev/null 2>gpurun_out/ncu_$k.err; echo $k rc=$?
done
