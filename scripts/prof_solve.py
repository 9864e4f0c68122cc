"""Profiling driver: one C3 solve of a fixed iteration count (for ncu -k ... --launch-skip)."""
import sys

sys.path.insert(0, ".")
import paper_2407_19689_b200 as pd  # noqa: E402

dp = pd.DeviceProblem.sqeuclid_grid(int(sys.argv[1]) if len(sys.argv) > 1 else 128, 0)
pd.solve_device(dp, pd.SolverConfig(tol=1e-12, max_iters=int(sys.argv[2]) if len(sys.argv) > 2 else 500))
