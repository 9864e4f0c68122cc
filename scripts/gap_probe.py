"""Measurement tooling: the K2 -> next K0 launch gap of the screened pass at C3 vs the
number of passes per CUDA-graph launch (poll_passes), from the device counters."""
import sys

sys.path.insert(0, ".")
import paper_2407_19689_b200 as pd  # noqa: E402

dp = pd.DeviceProblem.sqeuclid_grid(128, 0)
cfg = pd.SolverConfig(tol=1e-4)
(_, h), rep = pd.solve_device(dp, cfg)
for L in (4, 16, 64, 20, 4):
    h.screen_stats(reset=True)
    (_, h), rep = pd.solve_device(dp, cfg, handle=h, poll_passes=L)
    st = h.screen_stats()
    p = st["passes"]
    print(f"L={L:3d}: {rep._device_s * 1e3:7.2f} ms, pass {1e6 * rep._device_s / rep._passes:6.2f} us, "
          f"K2->K0 entry {st['gap_k2_k0_entry_ns'] / p / 1e3:5.2f} us, K2->K0 stamp {st['gap_k2_k0_ns'] / p / 1e3:5.2f}, "
          f"K0->K1 {st['k0_to_k1_ns'] / p / 1e3:5.2f}, K1->K2 {st['k1_to_k2_ns'] / p / 1e3:5.2f}", flush=True)
