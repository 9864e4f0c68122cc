"""Measurement tooling: the per-GPU work of an 8-GPU C5 run (65536^2), measured on one GPU.

Rank 0 of 8 owns rows 0..8191 of the 65536 x 65536 instance.  The screened pass of
that shard is timed by solving the row block as a standalone 8192 x 65536 problem
(rows of C generated on the device; its trajectory is not C5's, so this is a per-pass
cost probe, not a C5 solve), and by one dense 40 B/entry STEP pass over the block.
Prints one JSON line: screened pass time and K1 / K2 shares, dense STEP kernel time."""
import ctypes
import json
import sys

sys.path.insert(0, ".")
import paper_2407_19689_b200 as pd  # noqa: E402
from paper_2407_19689_b200 import _lib  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 400
dp = pd.DeviceProblem.sqeuclid_grid(256, 0, rows=(0, 8192))
cfg = pd.SolverConfig(tol=1e-12, max_iters=iters)
(_, h), rep = pd.solve_device(dp, cfg)
h.screen_stats(reset=True)
(_, h), rep = pd.solve_device(dp, cfg, handle=h)
st = h.screen_stats()
ms = ctypes.c_double()
_lib.check(h.lib.pdot_time_stream_kernel(h.ptr, 10, ctypes.byref(ms)))
p = max(1, st["passes"])
print(json.dumps({
    "shard": "rows 0..8191 of C5 (65536^2 sq-Euclidean, whitenoise seed 0), standalone solve",
    "iterations": rep.iterations, "passes": rep._passes, "device_s": rep._device_s,
    "pass_us_mean": 1e6 * rep._device_s / rep._passes, "k1_us": st["k1_ns"] / p / 1e3,
    "k2_us_to_last_block": st["k2_main_ns"] / p / 1e3, "k2_controller_us": st["k2_ctl_ns"] / p / 1e3,
    "active_cell_fraction": st["active_cells"] / (p * st["cells_per_plan"]),
    "k1_bytes_per_pass": st["k1_bytes"] / p,
    "dense_step_kernel_ms": ms.value, "dense_step_gbs": 40 * 8192 * 65536 / (ms.value * 1e-3) / 1e9}))
