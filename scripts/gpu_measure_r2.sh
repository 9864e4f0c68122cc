# Round-2 final measurement set for the current build (each ncu step only after
# the plain command exited 0): -m gpu suite, smoke, bench lines C1-C4 + the
# reference arm, pass timeline, screen trace, the ncu launch list of a short
# C3 bench, one --set full capture per screened-pass kernel at mid-solve, and
# K1's warm-cache DRAM traffic over a whole 600-iteration C3 solve.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f_suite.log 2>&1; echo suite rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/f_c3.json 2> gpurun_out/f_c3.err; echo c3 rc=$?
timeout 600 python bench.py --config c1 --no-cpu > gpurun_out/f_c1.json 2> gpurun_out/f_c1.err; echo c1 rc=$?
timeout 600 python bench.py --config c2 --no-cpu > gpurun_out/f_c2.json 2> gpurun_out/f_c2.err; echo c2 rc=$?
timeout 900 python bench.py --config c4 --no-cpu > gpurun_out/f_c4.json 2> gpurun_out/f_c4.err; echo c4 rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/f_ref.json 2> gpurun_out/f_ref.err; echo ref rc=$?
timeout 300 python scripts/k2_trace.py 128 400 > gpurun_out/f_k2trace.txt 2>&1
timeout 600 python scripts/screen_trace.py 128 1e-4 > gpurun_out/f_screen_trace.txt 2>&1
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-variant --no-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/f_launches.csv $B > /dev/null 2>gpurun_out/f_l.err; echo launches rc=$?
P="python scripts/prof_solve.py 128 500"
for k in unit_kernel screen_kernel tile_kernel finalize_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 300 --launch-count 1 -o gpurun_out/f_full_$k -f $P > /dev/null 2>gpurun_out/f_$k.err; echo $k rc=$?
done
python scripts/prof_solve.py 128 600 > gpurun_out/f_k1_alg.json 2>&1; echo alg rc=$?
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -k regex:unit_kernel --csv --log-file gpurun_out/f_k1_dram.csv python scripts/prof_solve.py 128 600 > /dev/null 2>gpurun_out/f_dram.err; echo dram rc=$?
