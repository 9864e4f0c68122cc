set -x
mkdir -p paper_2407_19689_b200/lib/variants
PDOT_NVCC_EXTRA="-DPDOT_K1_PROF" PDOT_BUILD_OUT=$PWD/paper_2407_19689_b200/lib/variants/k1prof.so python -c "from paper_2407_19689_b200.build import build_library; build_library(force=True)"
PDOT_LIB_PATH=$PWD/paper_2407_19689_b200/lib/variants/k1prof.so timeout 300 python scripts/prof_solve.py 128 700 > gpurun_out/zc_prof.txt 2>&1
bash scripts/gpu_ab_build.sh nozero=-DPDOT_K1_NO_ZERO_CELLS
python -m pytest tests/test_gpu_screen.py -x -q > gpurun_out/zc_tests.log 2>&1; tail -3 gpurun_out/zc_tests.log
