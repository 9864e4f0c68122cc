"""Measurement tooling: where the end-to-end C3 solve (host problem in pinned
memory -> numpy plan) spends its time."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_19689_b200 as pd  # noqa: E402
from paper_2407_19689_b200 import device, instances as inst  # noqa: E402

r = int(sys.argv[1]) if len(sys.argv) > 1 else 128
prob = inst.sqeuclid_problem(r, 0)
t = torch.empty(prob.C.shape, dtype=torch.float64, pin_memory=True)
t.numpy()[...] = prob.C
prob.cost.entries = t.numpy()
_ = prob.cost_fro_norm, prob.marginal_norm
cfg = pd.SolverConfig(tol=1e-4)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    it, rep_ = pd.solve(prob, cfg)
    t1 = time.perf_counter()
    print(f"solve {t1 - t0:.4f}s iters {rep_.iterations} phases " +
          " ".join(f"{k}={v:.4f}" for k, v in rep_._phases.items()), flush=True)
# pieces: the sparse copy of the final plan
(slot, hh), rep2 = pd.solve_device(device.DeviceProblem.from_host(prob), cfg)
import ctypes
from paper_2407_19689_b200 import _lib
import mmap
def zeros_small_pages(shape):
    nbytes = int(np.prod(shape)) * 8
    mm = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    mm.madvise(mmap.MADV_NOHUGEPAGE)
    return np.frombuffer(mm, dtype=np.float64).reshape(shape)
for k in range(4):
    X = np.zeros((prob.m, prob.n)) if k < 2 else zeros_small_pages((prob.m, prob.n))
    p = np.empty(prob.m); q = np.empty(prob.n); cells = ctypes.c_int64()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _lib.check(hh.lib.pdot_get_slot_sparse(hh.ptr, slot, X.ctypes.data, prob.n, p.ctypes.data, q.ctypes.data,
                                           ctypes.byref(cells)))
    t1 = time.perf_counter()
    print(f"sparse d2h {'np.zeros' if k < 2 else 'mmap 4K'} {t1 - t0:.4f}s cells {cells.value} ({cells.value * 1024 / 1e6:.1f} MB)")
# pieces
torch.cuda.synchronize()
t0 = time.perf_counter()
dp = device.DeviceProblem.from_host(prob)
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"from_host {t1 - t0:.4f}s")
t0 = time.perf_counter()
dev = torch.empty(prob.C.shape, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
t1 = time.perf_counter()
dev.copy_(torch.from_numpy(prob.C), non_blocking=True)
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"alloc {t1 - t0:.4f}s copy {t2 - t1:.4f}s ({prob.C.nbytes / (t2 - t1) / 1e9:.1f} GB/s)")
