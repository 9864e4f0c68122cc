import os
import sys
from pathlib import Path

# Pin BLAS threads before numpy loads: the reference's dot products go through
# multithreaded OpenBLAS and its trajectories depend on the thread count
# (SURVEY F7), so every oracle comparison runs single-threaded.
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

try:  # numpy may already be loaded by a pytest plugin: limit OpenBLAS at run time too
    import threadpoolctl

    _BLAS_LIMIT = threadpoolctl.threadpool_limits(limits=1, user_api="blas")
except ImportError:  # pragma: no cover
    _BLAS_LIMIT = None

ROOT = Path(__file__).resolve().parents[1]
for p in (str(ROOT), str(ROOT / "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libpdot.so")
