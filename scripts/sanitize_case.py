"""Small solves + unit calls for compute-sanitizer (memcheck / racecheck / synccheck)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_2407_19689_b200 as pd  # noqa: E402
from paper_2407_19689_b200 import instances as inst  # noqa: E402
from paper_2407_19689_b200.shard import solve_virtual  # noqa: E402

prob = inst.sqeuclid_problem(8, 1)  # 64 x 64
it, rep = pd.solve(prob, pd.SolverConfig(tol=1e-4))
print("solve", rep.iterations, rep.restarts, rep.termination_reason)
rng = np.random.default_rng(0)
p3 = pd.make_problem(rng.random((5, 7)), rng.random(5) + 0.1, rng.random(7) + 0.1)  # odd n, partial tiles
it3, rep3 = pd.solve(p3, pd.SolverConfig(tol=1e-6), trace=pd.SolveTrace(record_inner=True))
print("odd", rep3.iterations)
k = pd.kkt_error(p3, it3)
Xr = pd.round_to_feasible(p3, it3.X)
b = pd.stepsize_bound(it3, pd.pdhg_step(p3, it3, 0.1, 0.1), 2.0)
dp = pd.DeviceProblem.sqeuclid_grid(32, 0, implicit=True)
_, r4 = solve_virtual(dp, pd.SolverConfig(tol=1e-3), 2)
print("virtual", r4.iterations, "ok")
