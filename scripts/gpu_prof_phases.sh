# per-phase instrumented builds (PDOT_K1_PROF, PDOT_K2_PROF) on a 700-iteration C3
# solve, plus the K2 per-block trace of the in-tree build
set -x
mkdir -p gpurun_out paper_2407_19689_b200/lib/variants
for v in K1 K2; do
  PDOT_NVCC_EXTRA="-DPDOT_${v}_PROF" PDOT_BUILD_OUT=$PWD/paper_2407_19689_b200/lib/variants/prof$v.so \
    python -c "from paper_2407_19689_b200.build import build_library; build_library(force=True)" || exit 1
  PDOT_LIB_PATH=$PWD/paper_2407_19689_b200/lib/variants/prof$v.so timeout 300 python scripts/prof_solve.py 128 700 \
    > gpurun_out/ph_$v.txt 2>&1
done
timeout 300 python scripts/k2_trace.py 128 400 > gpurun_out/ph_k2trace.txt 2>&1
