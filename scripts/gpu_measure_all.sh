# Round measurement set: bench lines for every config, the reference arm, the
# ncu launch list of a short C3 bench, one --set full capture per screened-pass
# kernel, the warm DRAM traffic of K1 over a whole solve, and the device-side
# pass timeline.
set -x
timeout 900 python bench.py > gpurun_out/m_c3.json 2> gpurun_out/m_c3.err; echo c3 rc=$?
timeout 600 python bench.py --config c1 --no-cpu > gpurun_out/m_c1.json 2> gpurun_out/m_c1.err; echo c1 rc=$?
timeout 600 python bench.py --config c2 --no-cpu > gpurun_out/m_c2.json 2> gpurun_out/m_c2.err; echo c2 rc=$?
timeout 900 python bench.py --config c4 --no-cpu > gpurun_out/m_c4.json 2> gpurun_out/m_c4.err; echo c4 rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/m_ref.json 2> gpurun_out/m_ref.err; echo ref rc=$?
timeout 300 python scripts/k2_trace.py 128 400 > gpurun_out/m_k2trace.txt 2>&1
timeout 600 python scripts/screen_trace.py 128 1e-4 > gpurun_out/m_screen_trace.txt 2>&1
# K1 DRAM traffic of every launch of one deterministic 600-iteration solve (warm
# caches: --cache-control none), against the same solve's algorithmic bytes
timeout 300 python scripts/prof_solve.py 128 600 > gpurun_out/m_k1_alg.json 2> gpurun_out/m_k1_alg.err; echo alg rc=$?
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none -k regex:unit_kernel --csv --log-file gpurun_out/m_k1_dram.csv python scripts/prof_solve.py 128 600 > /dev/null 2>&1; echo dram rc=$?
B="python bench.py --steps 120 --warmup 5 --no-tol --no-e2e --no-variant --no-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/m_launches.csv $B > /dev/null 2>&1; echo ncu-list rc=$?
for k in unit_kernel screen_kernel tile_kernel finalize_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 90 --launch-count 1 -o gpurun_out/m_full_$k -f $B > /dev/null 2>&1; echo $k rc=$?
done
