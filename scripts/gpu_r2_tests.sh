# round-2 GPU check: new parity tests first (verbose), then the whole -m gpu suite and smoke
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/test_gpu_headline_parity.py tests/test_gpu_solve.py -q -s -k "${K:-.}" 2>&1 | tee gpurun_out/r2_parity.log | tail -60
timeout 1500 python -m pytest tests/ -q -m gpu -x ${EXTRA:-} 2>&1 | tee gpurun_out/r2_gpu_all.log | tail -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
