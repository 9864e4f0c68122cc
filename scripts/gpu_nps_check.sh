# next-pass screen in K2: a short bounded smoke first, then the screened-walker
# bit-identity suites, then an in-run A/B (PDOT_NPS=0 turns it off) on C3
set -x
mkdir -p gpurun_out
timeout 120 python scripts/prof_solve.py 128 100 > gpurun_out/nps_smoke.txt 2>&1; echo smoke rc=$?
tail -2 gpurun_out/nps_smoke.txt
timeout 900 python -m pytest tests/test_gpu_screen.py tests/test_gpu_slack_cert.py tests/test_gpu_pdl.py -x -q > gpurun_out/nps_tests.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/nps_tests.log
bash scripts/gpu_ab_envs.sh nonps=PDOT_NPS=0
