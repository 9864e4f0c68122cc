# slack certificates: screened-walker bit-identity suites, then an in-run A/B
# (PDOT_SREC=0 turns them off) on C3
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_screen.py tests/test_gpu_pdl.py -x -q > gpurun_out/sr_tests.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/sr_tests.log
bash scripts/gpu_ab_envs.sh nosr=PDOT_SREC=0
