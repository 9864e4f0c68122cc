"""Measurement tooling: does GPU idle time before a solve slow the solve loop?
C3 device-resident solves after sleeping s seconds (the e2e path leaves the
GPU idle during the host->device copy of C)."""
import sys
import time

sys.path.insert(0, ".")
import paper_2407_19689_b200 as pd  # noqa: E402

dp = pd.DeviceProblem.sqeuclid_grid(128, 0)
cfg = pd.SolverConfig(tol=1e-4)
(_, h), rep = pd.solve_device(dp, cfg)
for s in (0.0, 0.0, 0.02, 0.05, 0.1, 0.25, 0.5, 0.0, 1.0, 0.0):
    time.sleep(s)
    (_, h), rep = pd.solve_device(dp, cfg, handle=h)
    print(f"idle {s:5.2f} s -> loop device {rep._device_s * 1e3:7.2f} ms, wall {rep.wall_time_s * 1e3:7.2f} ms, "
          f"{rep.iterations} it", flush=True)
