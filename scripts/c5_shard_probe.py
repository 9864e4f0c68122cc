"""C5 (m = n = 65536) rank-0-of-8 shard on one GPU: build its 8192 x 65536 cost rows
on the device, run a short solve pass sequence through the virtual single-rank path,
and time the STEP kernel (explicit and matrix-free)."""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2407_19689_b200 as pd  # noqa: E402
from paper_2407_19689_b200 import _lib  # noqa: E402
from paper_2407_19689_b200.device import Handle  # noqa: E402
from paper_2407_19689_b200.shard import shard_rows  # noqa: E402

m = n = 65536
R = 8
r0, r1 = shard_rows(m, n, R, 0)
for implicit in (False, True):
    t0 = time.perf_counter()
    dp = pd.DeviceProblem.sqeuclid_grid(256, 0, rows=(r0, r1), implicit=implicit)
    h = Handle(m, n, 0, R, 0)
    h.bind(dp)
    build = time.perf_counter() - t0
    ms = ctypes.c_double()
    _lib.check(h.lib.pdot_time_stream_kernel(h.ptr, 10, ctypes.byref(ms)))
    bpe = 32 if implicit else 40
    gbs = bpe * (r1 - r0) * n / (ms.value * 1e-3) / 1e9
    print(f"C5 shard rows [{r0},{r1}) implicit={implicit}: build {build:.2f}s, step kernel {ms.value:.3f} ms "
          f"({gbs:.0f} GB/s at {bpe} B/elem); per-GPU pass estimate at 8 GPUs", flush=True)
    h.close()
    del dp
