"""Profiling driver: one C3 solve of a fixed iteration count (for ncu -k ... --launch-skip).

Prints the solve's screened-pass counters (one JSON line) so that ncu totals
over the same deterministic solve can be set against the algorithmic bytes.
"""
import json
import sys

sys.path.insert(0, ".")
import paper_2407_19689_b200 as pd  # noqa: E402

dp = pd.DeviceProblem.sqeuclid_grid(int(sys.argv[1]) if len(sys.argv) > 1 else 128, 0)
(_, h), rep = pd.solve_device(dp, pd.SolverConfig(tol=1e-12, max_iters=int(sys.argv[2]) if len(sys.argv) > 2 else 500))
st = h.screen_stats()
print(json.dumps({"passes_total": rep._passes, "iterations": rep.iterations, **st}))
