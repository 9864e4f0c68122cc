"""Measurement / validation tooling: C5 geometry at a larger row count.

Rows 0..8191 of the 65536 x 65536 C5 cost (generated on the device; 4.3 GB per
matrix) with the C5 column marginal and the rows' share of the row marginal
rescaled to unit mass (a balanced sub-problem), solved for a fixed number of
iterations on one handle and as 8 virtual row shards (device-copy exchange,
screened passes): the returned iterates must agree bit for bit.  Prints one JSON
line."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2407_19689_b200 as pd  # noqa: E402
from paper_2407_19689_b200.shard import solve_virtual  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
from paper_2407_19689_b200 import _lib  # noqa: E402
from paper_2407_19689_b200.instances import sqeuclid_fro_norm, whitenoise_marginals  # noqa: E402

f, g = whitenoise_marginals(256, 0)
fb = np.zeros_like(f)
fb[:rows] = f[:rows] / f[:rows].sum()
dp = pd.DeviceProblem.generated(_lib.COST_SQEUCLID_GRID, 65536, 65536, (256, 256, 0, 0), fb, g,
                                fro=sqeuclid_fro_norm(256), rows=(0, rows))
cfg = pd.SolverConfig(tol=1e-12, deterministic=True, max_iters=iters)
t0 = time.perf_counter()
it1, rep1 = pd.solve(dp, cfg)
t1 = time.perf_counter()
screened = pd.device.get_handle(dp.m, dp.n).screened()
pd.release_handles()
itv, repv = solve_virtual(dp, cfg, 8)
t2 = time.perf_counter()
same = (np.array_equal(itv.X, it1.X) and np.array_equal(itv.p, it1.p) and np.array_equal(itv.q, it1.q)
        and repv.iterations == rep1.iterations and repv.restart_lengths == rep1.restart_lengths)
print(json.dumps({"geometry": f"rows 0..{rows - 1} of C5 (n = 65536), {iters} iterations",
                  "screened": screened, "bit_identical_8_virtual_shards": bool(same),
                  "iterations": rep1.iterations, "restarts": rep1.restarts,
                  "nonzeros": int(np.count_nonzero(it1.X)), "single_s": t1 - t0, "virtual_s": t2 - t1}))
