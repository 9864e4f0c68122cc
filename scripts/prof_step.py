"""Short driver for ncu: C3 instance, a few solve iterations, then STEP kernels.

    python scripts/prof_step.py [--r 128] [--iters 30] [--kernel-launches 3]
"""
import argparse
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2407_19689_b200 as pd  # noqa: E402
from paper_2407_19689_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--r", type=int, default=128)
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--kernel-launches", type=int, default=3)
ap.add_argument("--implicit", action="store_true")
a = ap.parse_args()
dp = pd.DeviceProblem.sqeuclid_grid(a.r, 0, implicit=a.implicit)
(slot, h), rep = pd.solve_device(dp, pd.SolverConfig(tol=1e-12, max_iters=a.iters))
ms = ctypes.c_double()
import torch  # noqa: E402

torch.cuda.synchronize()
torch.cuda.profiler.start()  # ncu --profile-from-start off captures only the STEP launches below
_lib.check(h.lib.pdot_time_stream_kernel(h.ptr, a.kernel_launches, ctypes.byref(ms)))
torch.cuda.profiler.stop()
res = _lib.Result()
_lib.check(h.lib.pdot_resume(h.ptr, a.iters + 100, ctypes.byref(res)))
per_pass = res.device_s / (res.passes - rep._passes)
msf = ctypes.c_double()
_lib.check(h.lib.pdot_time_finalize(h.ptr, 50, ctypes.byref(msf)))
print(f"finalize {msf.value * 1e3:.1f} us; solve pass {per_pass * 1e3:.4f} ms, overhead/pass "
      f"{(per_pass * 1e3 - ms.value) * 1e3:.1f} us")
print(f"iters {rep.iterations} passes {rep._passes} step-kernel {ms.value:.3f} ms "
      f"-> {40 * a.r**4 / ms.value / 1e6:.0f} GB/s")
