import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2407_19689_b200 as pd  # noqa: E402
dp = pd.DeviceProblem.sqeuclid_grid(128, 0)
for iters in (10, 110):
    _, _, rep = pd.sinkhorn_solve(dp, pd.SinkhornConfig(penalty=1.0, tol=1e-12, max_iters=iters), poll_iters=50)
    print(iters, rep.iterations, rep.wall_time_s, rep.termination_reason, flush=True)
