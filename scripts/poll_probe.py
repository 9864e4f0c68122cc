"""Measurement tooling: C3 time-to-1e-4 (solve_device, report.wall_time_s) against the
number of passes per graph launch (poll_passes; 0 = auto_batch)."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2407_19689_b200 as pd  # noqa: E402

r = int(sys.argv[1]) if len(sys.argv) > 1 else 128
dp = pd.DeviceProblem.sqeuclid_grid(r, 0)
cfg = pd.SolverConfig(tol=1e-4)
pd.solve_device(dp, cfg)  # warm-up (handle, graph, clocks)
for L in (0, 8, 12, 32, 48, 64, 0):
    ts = []
    for _ in range(5):
        (_, h), rep = pd.solve_device(dp, cfg, poll_passes=L)
        ts.append(rep.wall_time_s)
    print(f"poll_passes {L:3d}: wall {np.median(ts) * 1e3:.2f} ms (min {min(ts) * 1e3:.2f}), "
          f"{rep.iterations} it, {rep.iterations / np.median(ts):.0f} iter/s", flush=True)
