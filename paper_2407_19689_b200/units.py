"""Unit entry points with the reference signatures, each one CUDA pass.

These are the functions the reference tests call directly:
``pdhg_step`` (pdhg.py:121-129), ``stepsize_bound`` (pdhg.py:132-149),
``adaptive_stepsize`` (pdhg.py:152-171), ``kkt_error`` (kkt.py:56-94),
``duality_gap`` (kkt.py:97-101), ``restart_candidate`` (pdhg.py:189-195),
``apply_A`` / ``apply_At`` (operator.py:36-43) and ``round_to_feasible``
(rounding.py:18-40).  Inputs and outputs are numpy, as in the reference; the
arithmetic runs in libpdot.so on the GPU (the same streaming/finalize kernels
the solve loop uses).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .config import eta_from_bound
from .device import DeviceProblem, as_device_problem, get_handle, require_cuda, torch
from .records import Iterate, KKTReport


def _out(n):
    return (ctypes.c_double * n)()


def _bound_handle(prob):
    dp = as_device_problem(prob)
    h = get_handle(dp.m, dp.n, dp.device)
    h.bind(dp)
    return dp, h


def apply_A(X: np.ndarray):
    """Row sums and column sums of the plan (operator.py:36-38)."""
    X = np.asarray(X, dtype=np.float64)
    m, n = X.shape
    h = get_handle(m, n)
    h.set_slot(0, X, None, None)
    rows, cols = np.empty(m), np.empty(n)
    _lib.check(h.lib.pdot_unit_apply_A(h.ptr, rows.ctypes.data, cols.ctypes.data))
    return rows, cols


def apply_At(p: np.ndarray, q: np.ndarray) -> np.ndarray:
    """Adjoint of the constraint map: entry (i, j) is p_i + q_j (operator.py:41-43)."""
    require_cuda()
    p = np.ascontiguousarray(p, dtype=np.float64)
    q = np.ascontiguousarray(q, dtype=np.float64)
    m, n = p.size, q.size
    pt = torch.from_numpy(p).cuda()
    qt = torch.from_numpy(q).cuda()
    out = torch.empty((m, n), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    _lib.check(_lib.load().pdot_apply_At(pt.data_ptr(), qt.data_ptr(), m, n, out.data_ptr(), n))
    return out.cpu().numpy()


def pdhg_step(prob, it: Iterate, tau: float, sigma: float) -> Iterate:
    """One primal-dual step (pdhg.py:121-129) on the GPU."""
    dp, h = _bound_handle(prob)
    h.set_slot(0, it.X, it.p, it.q)
    _lib.check(h.lib.pdot_unit_step(h.ptr, float(tau), float(sigma), 0.0))
    X, p, q = h.get_slot(1)
    return Iterate(X, p, q)


def step_and_average(prob, it: Iterate, avg: Iterate, tau: float, sigma: float, k: int):
    """One fused STEP pass as the solve loop runs it: the trial ``next =
    pdhg_step(it)`` plus the running-mean updates of pdhg.py:314-317 with count
    k -- the average MATRIX of the input iterate, ``avg.X + (it.X - avg.X)/k``
    (computed one pass late in the loop), and the average DUALS of the trial,
    ``avg.p + (next.p - avg.p)/k``.  Returns (next, new_average)."""
    if k < 1:
        raise ValueError("k must be >= 1")
    dp, h = _bound_handle(prob)
    h.set_slot(0, it.X, it.p, it.q)
    h.set_slot(2, avg.X, avg.p, avg.q)
    h.set_slot(3, None, avg.p, avg.q)
    _lib.check(h.lib.pdot_unit_step(h.ptr, float(tau), float(sigma), float(k)))
    X, p, q = h.get_slot(1)
    A, pa, qa = h.get_slot(3)
    return Iterate(X, p, q), Iterate(A, pa, qa)


def stepsize_bound(it: Iterate, it_next: Iterate, omega: float, eps_zero: float = 1e-10) -> float:
    """Largest admissible step-size scale for the displacement (pdhg.py:132-149)."""
    m, n = np.shape(it.X)
    h = get_handle(m, n)
    h.set_slot(0, it.X, it.p, it.q)
    h.set_slot(1, it_next.X, it_next.p, it_next.q)
    out = _out(5)
    _lib.check(h.lib.pdot_unit_bound(h.ptr, float(omega), float(eps_zero), out))
    return float(out[0])


def adaptive_stepsize(it: Iterate, it_next: Iterate, omega: float, eta_current: float,
                      eps_zero: float = 1e-10) -> float:
    """Halve eta until it satisfies the bound, then grow 1.05x capped (pdhg.py:152-171)."""
    return eta_from_bound(stepsize_bound(it, it_next, omega, eps_zero), eta_current)


def _kkt(prob, it: Iterate, scale_R: float, want_arrays: bool):
    if scale_R <= 0:
        raise ValueError("scale_R must be positive")
    dp, h = _bound_handle(prob)
    h.set_slot(0, it.X, it.p, it.q)
    m, n = dp.m, dp.n
    viol = np.empty((m, n)) if want_arrays else None
    rows, cols = np.empty(m), np.empty(n)
    out = _out(10)
    _lib.check(h.lib.pdot_unit_kkt(h.ptr, float(scale_R), viol.ctypes.data if want_arrays else None, n,
                                   rows.ctypes.data, cols.ctypes.data, out))
    return out, rows, cols, viol


def _host_marginals(prob):
    if isinstance(prob, DeviceProblem):
        if prob.host is not None:
            return np.asarray(prob.host.f), np.asarray(prob.host.g)
        return prob.f_t.cpu().numpy(), prob.g_t.cpu().numpy()
    return np.asarray(prob.f), np.asarray(prob.g)


def kkt_error(prob, it: Iterate, scale_R: float = 1.0) -> KKTReport:
    """All KKT residual blocks, matrix-free, on the GPU (kkt.py:56-94)."""
    out, rows, cols, viol = _kkt(prob, it, scale_R, True)
    f, g = _host_marginals(prob)
    return KKTReport(primal_row=rows - f, primal_col=cols - g, dual_violation=viol, gap=float(out[0]),
                     scale_R=float(scale_R), composite=float(out[1]), relative_composite=float(out[2]))


def duality_gap(prob, it: Iterate) -> float:
    """|<C, X> - f.p - g.q| (kkt.py:97-101)."""
    out, _, _, _ = _kkt(prob, it, 1.0, False)
    return abs(float(out[0]))


def restart_candidate(current: Iterate, average: Iterate, prob, scale_R: float) -> Iterate:
    """The current iterate if its relative KKT is strictly smaller, else the average (pdhg.py:189-195)."""
    kc = _kkt(prob, current, scale_R, False)[0][2]
    ka = _kkt(prob, average, scale_R, False)[0][2]
    return current if kc < ka else average


def round_to_feasible(prob, X: np.ndarray) -> np.ndarray:
    """Algorithm-3 rounding to an exactly feasible plan (rounding.py:18-40) on the GPU."""
    dp, h = _bound_handle(prob)
    h.set_slot(0, X, None, None)
    Xf = np.empty((dp.m, dp.n))
    out = _out(3)
    _lib.check(h.lib.pdot_round(h.ptr, 0, Xf.ctypes.data, dp.n, out))
    return Xf


def rounded_objective(prob, X: np.ndarray) -> float:
    """<C, round_to_feasible(X)> without materialising X_feas on the host."""
    dp, h = _bound_handle(prob)
    h.set_slot(0, X, None, None)
    out = _out(3)
    _lib.check(h.lib.pdot_round(h.ptr, 0, None, 0, out))
    return float(out[0])


def rounding_bound_check(prob, X: np.ndarray, X_feas: np.ndarray) -> bool:
    """Lemma 2 of the paper: |X_feas - X|_1 <= 2 (|f - X 1|_1 + |g - X^T 1|_1)
    (rounding.py:43-50, same slack 1e-12 (1 + rhs)).  The marginal residuals
    come from the GPU row / column sums; the entrywise l1 distance is reduced
    on the device."""
    require_cuda()
    f, g = _host_marginals(prob)
    rows, cols = apply_A(X)
    rhs = 2.0 * (float(np.abs(f - rows).sum()) + float(np.abs(g - cols).sum()))
    a = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float64)).cuda()
    b = torch.from_numpy(np.ascontiguousarray(X_feas, dtype=np.float64)).cuda()
    lhs = float((b - a).abs().sum().item())
    return lhs <= rhs + 1e-12 * (1.0 + rhs)
