"""Large-instance check (not a test: 8.6 GB per matrix): a 32768^2 solve of a
fixed iteration count with screening on and off must agree bit for bit, and
the screened pass must exercise the multi-wave finalize grid."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2407_19689_b200 as pd  # noqa: E402
from paper_2407_19689_b200 import device  # noqa: E402

r = int(sys.argv[1]) if len(sys.argv) > 1 else 256
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 120
dp = pd.DeviceProblem.sqeuclid_grid(r, 0)
out = []
for on in (False, True):
    device.set_screening(on)
    (slot, h), rep = pd.solve_device(dp, pd.SolverConfig(tol=1e-12, max_iters=iters, deterministic=True))
    X, p, q = h.get_slot(slot)
    out.append((rep.to_json(), X.view(np.int64).sum(dtype=np.int64), p.copy(), q.copy(), rep._passes))
    print("screen", on, "iters", rep.iterations, "passes", rep._passes, "kkt", rep.final_relative_kkt, flush=True)
    del X
same = out[0][0] == out[1][0] and out[0][1] == out[1][1] and np.array_equal(out[0][2].view(np.int64), out[1][2].view(np.int64)) \
    and np.array_equal(out[0][3].view(np.int64), out[1][3].view(np.int64))
print("m = n =", dp.m, "bit-identical:", same)
