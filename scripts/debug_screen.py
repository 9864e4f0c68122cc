"""Debug helper: step a screened solve one pass at a time (CUDA_LAUNCH_BLOCKING=1)."""
import ctypes
import sys

sys.path.insert(0, ".")
import paper_2407_19689_b200 as pd  # noqa: E402
from paper_2407_19689_b200 import _lib, device  # noqa: E402
from paper_2407_19689_b200 import instances as inst  # noqa: E402
from paper_2407_19689_b200.engine import config_struct  # noqa: E402

r = int(sys.argv[1]) if len(sys.argv) > 1 else 8
dp = pd.DeviceProblem.from_host(inst.sqeuclid_problem(r, 1))
h = device.get_handle(dp.m, dp.n, dp.device)
h.bind(dp)
h.set_screening(True)
h.set_slot(0, None, None, None)
cfg = config_struct(pd.SolverConfig(tol=1e-6), trace_level=0)
_lib.check(h.lib.pdot_begin(h.ptr, ctypes.byref(cfg), 0.0))
prog = _lib.Progress()
for k in range(100000):
    op_before = prog.op
    try:
        _lib.check(h.lib.pdot_advance(h.ptr, 1, ctypes.byref(prog)))
    except RuntimeError as e:
        print("FAILED at pass", k, "op(before)", op_before, e)
        raise
    if k < 5 or k % 100 == 0:
        print("pass", k, "op", prog.op, "it", prog.iterations, flush=True)
    if prog.done:
        print("done", prog.iterations)
        break
