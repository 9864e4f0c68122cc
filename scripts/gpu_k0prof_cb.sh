# K0 phase profile (PDOT_K0_PROF) and an A/B of K2's column batch (PDOT_COL_BATCH 3, 4)
set -x
mkdir -p gpurun_out paper_2407_19689_b200/lib/variants
PDOT_NVCC_EXTRA="-DPDOT_K0_PROF" PDOT_BUILD_OUT=$PWD/paper_2407_19689_b200/lib/variants/profK0.so \
  python -c "from paper_2407_19689_b200.build import build_library; build_library(force=True)"
PDOT_LIB_PATH=$PWD/paper_2407_19689_b200/lib/variants/profK0.so timeout 300 python scripts/prof_solve.py 128 700 > gpurun_out/ph_K0.txt 2>&1
bash scripts/gpu_ab_build.sh cb3=-DPDOT_COL_BATCH=3 cb4=-DPDOT_COL_BATCH=4
