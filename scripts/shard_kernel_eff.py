"""STEP-kernel time of ONE row shard of C3 (the per-GPU work at R GPUs), on one GPU."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2407_19689_b200 as pd  # noqa: E402
from paper_2407_19689_b200 import _lib  # noqa: E402
from paper_2407_19689_b200.device import Handle  # noqa: E402
from paper_2407_19689_b200.shard import shard_rows  # noqa: E402

m = n = 16384
for R in (1, 2, 4, 8):
    r0, r1 = shard_rows(m, n, R, 0)
    dp = pd.DeviceProblem.sqeuclid_grid(128, 0, rows=(r0, r1))
    h = Handle(m, n, 0, R, 0)
    h.bind(dp)
    ms = ctypes.c_double()
    _lib.check(h.lib.pdot_time_stream_kernel(h.ptr, 30, ctypes.byref(ms)))
    ideal = 1.645 / R
    print(f"R={R}: rows {r1 - r0}, step kernel {ms.value:.4f} ms, ideal {ideal:.4f} ms, eff {ideal / ms.value:.3f}")
    h.close()
    del dp
