"""Measurement tooling: R row shards of C3 (16384^2, screened passes) stepped on ONE
GPU as virtual shards (device-copy exchange), for the per-shard latency model of
DESIGN.md §6.  Run under ncu (gpu__time_duration per launch) and parse with
scripts/shard_model.py; launch order per pass: for each shard K0 screen_kernel,
K1 unit_kernel, K1b tile_kernel, K2a finalize_kernel; then K2b finalize_kernel
of every shard.  No kernel waits on another (the exchange is a host-ordered copy).

    python scripts/shard_probe.py R PASSES
"""
import ctypes
import sys

sys.path.insert(0, ".")
import paper_2407_19689_b200 as pd  # noqa: E402
from paper_2407_19689_b200 import _lib  # noqa: E402
from paper_2407_19689_b200.device import Handle  # noqa: E402
from paper_2407_19689_b200.engine import config_struct  # noqa: E402

R, passes = int(sys.argv[1]), int(sys.argv[2])
dp = pd.DeviceProblem.sqeuclid_grid(128, 0)
hs = [Handle(dp.m, dp.n, 0, R, r) for r in range(R)]
for h in hs:
    h.bind(dp.row_shard(h.row0, h.row0 + h.m))
    _lib.check(h.lib.pdot_set_virtual(h.ptr, 1))
    h.set_slot(0, None, None, None)
arr = (ctypes.c_void_p * R)(*[h.ptr.value for h in hs])
cfg = config_struct(pd.SolverConfig(tol=1e-12), trace_level=0)
for h in hs:
    _lib.check(h.lib.pdot_begin(h.ptr, ctypes.byref(cfg), 0.0))
prog = _lib.Progress()
lib = hs[0].lib
ms = (ctypes.c_double * 2)()
t = [0.0, 0.0]
for k in range(passes):
    for h in hs:
        _lib.check(lib.pdot_shard_pass(h.ptr, 0, None))
    _lib.check(lib.pdot_exchange_local(arr, R))
    for h in hs:
        _lib.check(lib.pdot_shard_pass(h.ptr, 1, ctypes.byref(prog)))
print(f"R={R}: {passes} passes, {prog.iterations} iterations, {prog.restarts} restarts", flush=True)
