"""Per-pass screening statistics of one solve (measurement tooling).

Steps the solve one pass at a time (pdot_advance) and records, per pass, the
active 8x16 cells, the tiles K1 visited, the bytes K1 moved and the K1
duration (%globaltimer).  Usage: python scripts/screen_trace.py R [tol] [max_passes]
"""
import ctypes
import json
import sys

sys.path.insert(0, ".")
import paper_2407_19689_b200 as pd  # noqa: E402
from paper_2407_19689_b200 import _lib, device  # noqa: E402
from paper_2407_19689_b200.engine import config_struct  # noqa: E402

r = int(sys.argv[1])
tol = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-4
max_passes = int(sys.argv[3]) if len(sys.argv) > 3 else 100000
dp = pd.DeviceProblem.sqeuclid_grid(r, 0)
h = device.get_handle(dp.m, dp.n, dp.device)
h.bind(dp)
h.set_slot(0, None, None, None)
cfg = config_struct(pd.SolverConfig(tol=tol), trace_level=0)
_lib.check(h.lib.pdot_begin(h.ptr, ctypes.byref(cfg), 0.0))
prog = _lib.Progress()
h.screen_stats(reset=True)
prev = h.screen_stats()
rows = []
for k in range(max_passes):
    _lib.check(h.lib.pdot_advance(h.ptr, 1, ctypes.byref(prog)))
    st = h.screen_stats()
    d = {key: st[key] - prev[key] for key in ("passes", "active_cells", "cells_visited", "k1_bytes", "k1_ns", "k2_main_ns", "k2_ctl_ns", "ctl_reduce_ns", "ctl_logic_ns", "ctl_publish_ns")}
    prev = st
    d["it"] = prog.iterations
    d["frac"] = d["active_cells"] / st["cells_per_plan"]
    rows.append(d)
    if prog.done:
        break
res = _lib.Result()
_lib.check(h.lib.pdot_finish(h.ptr, ctypes.byref(res)))
steps = [x for x in rows if x["passes"]]
summary = {"r": r, "iterations": res.iterations, "passes": len(rows),
           "mean_frac": sum(x["frac"] for x in steps) / len(steps),
           "mean_k1_us": sum(x["k1_ns"] for x in steps) / len(steps) / 1e3,
           "mean_cells_visited": sum(x["cells_visited"] for x in steps) / len(steps),
           "mean_k2_main_us": sum(x["k2_main_ns"] for x in steps) / len(steps) / 1e3,
           "mean_k2_ctl_us": sum(x["k2_ctl_ns"] for x in steps) / len(steps) / 1e3,
           "mean_ctl_reduce_us": sum(x["ctl_reduce_ns"] for x in steps) / len(steps) / 1e3,
           "mean_ctl_logic_us": sum(x["ctl_logic_ns"] for x in steps) / len(steps) / 1e3,
           "mean_ctl_publish_us": sum(x["ctl_publish_ns"] for x in steps) / len(steps) / 1e3,
           "mean_k1_MB": sum(x["k1_bytes"] for x in steps) / len(steps) / 1e6}
print(json.dumps(summary))
for i in range(0, len(rows), max(1, len(rows) // 60)):
    x = rows[i]
    print(i, x["it"], "frac %.4f cells %d MB %.1f K1 us %.1f K2 us %.1f + %.1f" % (
        x["frac"], x["cells_visited"], x["k1_bytes"] / 1e6, x["k1_ns"] / 1e3, x["k2_main_ns"] / 1e3, x["k2_ctl_ns"] / 1e3))
