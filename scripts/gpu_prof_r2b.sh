# Round-2 evidence for the CURRENT build: launch list, --set full of each screened-pass
# kernel at mid-solve, and K1's warm-cache DRAM traffic over a whole 600-iteration C3
# solve (ncu --cache-control none) against the same solve's algorithmic K1 bytes.
set -x
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-variant --no-cpu"
$B > gpurun_out/p2_plain.json 2>gpurun_out/p2_plain.err; echo plain rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/p2_launches.csv $B > /dev/null 2>gpurun_out/p2_l.err; echo launches rc=$?
P="python scripts/prof_solve.py 128 500"
for k in unit_kernel screen_kernel tile_kernel finalize_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 300 --launch-count 1 -o gpurun_out/p2_full_$k -f $P > /dev/null 2>gpurun_out/p2_$k.err; echo $k rc=$?
done
python scripts/prof_solve.py 128 600 > gpurun_out/p2_k1_alg.json 2>&1; echo alg rc=$?
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -k regex:unit_kernel --csv --log-file gpurun_out/p2_k1_dram.csv python scripts/prof_solve.py 128 600 > /dev/null 2>gpurun_out/p2_dram.err; echo dram rc=$?
