for v in s6_b1 s3_b2; do
export PDOT_LIB=paper_2407_19689_b200/lib/libpdot_$v.so
python scripts/prof_step.py --iters 5 --kernel-launches 1 > gpurun_out/prof2_plain_$v.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:stream_kernel -s 1 -c 1 -o gpurun_out/prof_step_tma_$v python scripts/prof_step.py --iters 5 --kernel-launches 1 > gpurun_out/ncu2_$v.log 2>&1
echo rc=$?
done
