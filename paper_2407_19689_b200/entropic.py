"""Log-domain Sinkhorn baseline on the GPU.

Same API as the reference's sinkhorn module (sinkhorn.py:25-150):
``SinkhornConfig``, ``Potentials``, ``sinkhorn_solve(prob, cfg) -> (plan,
Potentials, SolveReport)`` and ``sinkhorn_report_gap``.  The alternating
log-sum-exp potential updates stream C twice per iteration in
csrc/sinkhorn.cu; the final plan, its rounding and the rounded objective are
computed on the device as well.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import asdict, dataclass

import numpy as np

from . import _lib
from .device import as_device_problem, get_handle
from .records import SolveReport


@dataclass
class SinkhornConfig:
    penalty: float = 0.001
    tol: float = 1e-4
    max_iters: int = 100_000
    time_limit_s: float = 3600.0
    deterministic: bool = False

    def __post_init__(self):  # sinkhorn.py:33-37
        if self.penalty <= 0:
            raise ValueError("penalty must be positive")
        if self.tol <= 0 or self.max_iters < 1 or self.time_limit_s <= 0:
            raise ValueError("tol, max_iters and time_limit_s must be positive")


@dataclass(eq=False)
class Potentials:
    phi: np.ndarray
    psi: np.ndarray


def sinkhorn_solve(prob, cfg: SinkhornConfig | None = None, *, device: int = 0, poll_iters: int = 0):
    """Iterate until the l1 marginal violation of the plan is at most tol.

    Returns the (unrounded) plan, the dual potentials and a report whose
    objective and gap are evaluated on the rounded plan; ``final_relative_kkt``
    holds the terminal l1 feasibility (sinkhorn.py:58-130).
    """
    t0 = time.perf_counter()
    if cfg is None:
        cfg = SinkhornConfig()
    dp = as_device_problem(prob, device)
    if dp.implicit:
        raise ValueError("sinkhorn needs an explicit cost matrix")
    h = get_handle(dp.m, dp.n, dp.device)
    h.bind(dp)
    c = _lib.SinkhornCfg(penalty=cfg.penalty, tol=cfg.tol, max_iters=int(cfg.max_iters),
                         time_limit_s=cfg.time_limit_s, poll_iters=poll_iters)
    res = _lib.Result()
    _lib.check(h.lib.pdot_sinkhorn_solve(h.ptr, ctypes.byref(c), time.perf_counter() - t0, ctypes.byref(res)))
    elapsed = time.perf_counter() - t0
    # the plan sits in slot 0 (X) with the potentials as its (p, q)
    rows, cols = np.empty(dp.m), np.empty(dp.n)
    _lib.check(h.lib.pdot_unit_apply_A(h.ptr, rows.ctypes.data, cols.ctypes.data))
    f, g = (dp.f_t.cpu().numpy(), dp.g_t.cpu().numpy())
    feasibility = float(np.abs(rows - f).sum() + np.abs(cols - g).sum())  # sinkhorn.py:111-113
    out = (ctypes.c_double * 3)()
    _lib.check(h.lib.pdot_round(h.ptr, 0, None, 0, out))
    rounded, dual = float(out[0]), float(out[1])
    plan, phi, psi = h.get_slot(0)
    reason = _lib.REASONS.get(res.reason, "unknown")
    report = SolveReport(method="sinkhorn", solved=reason == "tolerance",
                         wall_time_s=0.0 if cfg.deterministic else float(elapsed),
                         iterations=int(res.iterations), restarts=0, final_relative_kkt=feasibility,
                         rounded_objective=rounded, duality_gap=abs(rounded - dual),
                         termination_reason=reason, config_echo=asdict(cfg))
    return plan, Potentials(phi, psi), report


def sinkhorn_report_gap(prob, plan: np.ndarray, potentials: Potentials, dual_bound: float | None = None) -> float:
    """Duality gap of the rounded plan against `dual_bound` or the potentials (sinkhorn.py:133-150)."""
    from .units import rounded_objective
    objective = rounded_objective(prob, plan)
    if dual_bound is None:
        dual_bound = float(np.asarray(prob.f) @ potentials.phi + np.asarray(prob.g) @ potentials.psi)
    return abs(objective - dual_bound)
