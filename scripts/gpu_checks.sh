# Correctness tooling on the GPU box:
#  1. the PDOT_DEVICE_CHECKS build (DCHECK traps on cell-list / band / cell / partial
#     index violations in the screened walkers) over the screened-walker test suite;
#  2. compute-sanitizer memcheck / racecheck / synccheck on small solves that take the
#     screened pass sequence, the dense walker, unit calls, rounding and virtual shards.
set -x
mkdir -p gpurun_out
OUT=$PWD/paper_2407_19689_b200/lib_checks/libpdot.so
PDOT_DEVICE_CHECKS=1 PDOT_BUILD_OUT=$OUT python -c "from paper_2407_19689_b200.build import build_library; print(build_library(force=True))"
PDOT_LIB_PATH=$OUT timeout 900 python -m pytest tests/test_gpu_screen.py tests/test_gpu_shard.py -m gpu -q 2>&1 | tail -5
for tool in memcheck racecheck synccheck; do
  PDOT_SCREEN=1 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_case.py 2>&1 | tail -6
  echo "$tool exit=${PIPESTATUS[0]}"
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_case.py 2>&1 | tail -4
  echo "$tool (default walkers) exit=${PIPESTATUS[0]}"
done
