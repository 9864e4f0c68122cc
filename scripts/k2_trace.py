"""Debug tooling: per-block K2 timeline of the last screened STEP pass (PDOT_K2_TRACE=1)."""
import ctypes
import os
import sys

os.environ["PDOT_K2_TRACE"] = "1"
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2407_19689_b200 as pd  # noqa: E402
from paper_2407_19689_b200 import _lib, device  # noqa: E402

dp = pd.DeviceProblem.sqeuclid_grid(int(sys.argv[1]) if len(sys.argv) > 1 else 128, 0)
it = int(sys.argv[2]) if len(sys.argv) > 2 else 400
(_, h), rep = pd.solve_device(dp, pd.SolverConfig(tol=1e-12, max_iters=5))
h.screen_stats(reset=True)
(_, h), rep = pd.solve_device(dp, pd.SolverConfig(tol=1e-12, max_iters=it))
lib = _lib.load()
lib.pdot_debug_k2.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int64]
buf = (ctypes.c_ulonglong * 8192)()
nb = lib.pdot_debug_k2(h.ptr, buf, 8192)
tl = np.array(buf[nb * 4 + 8:nb * 4 + 16], dtype=np.float64)
t00 = tl[0]
names = ("K0", "K1", "K1b", "K2")
print("pass timeline (us from K0 start): " + ", ".join(
    f"{names[k]} {(tl[2 * k] - t00) / 1e3:.1f}..{(tl[2 * k + 1] - t00) / 1e3:.1f}" for k in range(4)
    if 0 < tl[2 * k + 1] and tl[2 * k] < 2 ** 63))
a = np.array(buf[:nb * 4], dtype=np.float64).reshape(nb, 4)
t0 = a[:, 0].min()
a[:, :3] -= t0
T = dp.m // 128
print("blocks", nb, "row blocks", T)
for name, sl in (("row", slice(0, T)), ("column", slice(T, nb))):
    x = a[sl]
    print(f"{name}: entry {x[:,0].min():.0f}..{x[:,0].max():.0f} ns, work {np.median(x[:,1]-x[:,0]):.0f} "
          f"(max {(x[:,1]-x[:,0]).max():.0f}) ns, ticket at {x[:,2].min():.0f}..{x[:,2].max():.0f} ns")
st = h.screen_stats()
p = max(1, st["passes"])
print("per pass: K1 %.1f us, K2 to last ticket %.1f us, controller %.1f us (reduce %.1f, decide %.1f, publish %.1f)" % (
    st["k1_ns"] / p / 1e3, st["k2_main_ns"] / p / 1e3, st["k2_ctl_ns"] / p / 1e3, st["ctl_reduce_ns"] / p / 1e3,
    st["ctl_logic_ns"] / p / 1e3, st["ctl_publish_ns"] / p / 1e3))
z = list(buf[nb * 4 + 25:nb * 4 + 30])
if z[0]:
    print("K0 full-tile warp: start %.2f us, first-chunk load latency cold %d ns, warm %d ns, end %.2f us" % ((z[0] - buf[nb * 4 + 8]) / 1e3, z[1], z[2], (z[4] - buf[nb * 4 + 8]) / 1e3))
kb = list(buf[nb * 4 + 25:nb * 4 + 29])
if kb[0]:
    print("K1b: tiles %d, slowest list read %.2f us, columns max %.2f, rows phase max %.2f us, scalars phase max %.2f us" % (kb[0], kb[1] / 1e3, buf[nb * 4 + 29] / 1e3, kb[2] / 1e3, kb[3] / 1e3))
if os.environ.get("K2_COLSPLIT"):
    x = a[T:nb]
    x3 = x[:, 3] - t0
    print("column blocks: column sums done at median %.0f ns after entry (max %.0f), work end %.0f" % (
        np.median(x3 - x[:, 0]), (x3 - x[:, 0]).max(), np.median(x[:, 1] - x[:, 0])))
