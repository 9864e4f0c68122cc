"""CPU oracle for the log-domain Sinkhorn baseline — TEST INFRASTRUCTURE ONLY.

Restates the reference's sinkhorn_solve (/root/reference/pkg/src/otsolve/
sinkhorn.py:46-130) with the same numpy/scipy operations, so it reproduces the
reference bit for bit (pinned by tests/test_oracle_golden.py against fixtures
the reference produced).  Used only by tests/ and the CPU legs of bench.py.
"""

from __future__ import annotations

import time

import numpy as np
from scipy.special import logsumexp

from .pdot_oracle import feasible_rounding


def _potential_rows(psi, C, log_f, eps):  # sinkhorn.py:50-51
    return eps * log_f - eps * logsumexp((psi[None, :] - C) / eps, axis=1)


def _potential_cols(phi, C, log_g, eps):  # sinkhorn.py:54-55
    return eps * log_g - eps * logsumexp((phi[:, None] - C) / eps, axis=0)


def _plan(phi, psi, C, eps):  # sinkhorn.py:46-47
    return np.exp((phi[:, None] + psi[None, :] - C) / eps)


def oracle_sinkhorn(prob, penalty, tol, max_iters=100_000, time_limit_s=3600.0, clock=time.perf_counter):
    """sinkhorn.py:58-130.  Returns (plan, phi, psi, report_dict)."""
    t0 = clock()
    eps = penalty
    rmask, cmask = prob.f > 0, prob.g > 0
    f, g = prob.f[rmask], prob.g[cmask]
    C = prob.C[np.ix_(rmask, cmask)]
    log_f, log_g = np.log(f), np.log(g)
    phi, psi = np.zeros(f.size), np.zeros(g.size)
    it = 0
    reason = None
    X = _plan(phi, psi, C, eps)
    feas = float(np.abs(X.sum(axis=1) - f).sum() + np.abs(X.sum(axis=0) - g).sum())
    while reason is None:
        if it >= max_iters:
            reason = "iteration_limit"
            break
        if clock() - t0 > time_limit_s:
            reason = "time_limit"
            break
        phi = _potential_rows(psi, C, log_f, eps)
        psi = _potential_cols(phi, C, log_g, eps)
        it += 1
        if not (np.all(np.isfinite(phi)) and np.all(np.isfinite(psi))):
            raise RuntimeError("numerical failure: non-finite potential")
        X = _plan(phi, psi, C, eps)
        feas = float(np.abs(X.sum(axis=1) - f).sum() + np.abs(X.sum(axis=0) - g).sum())
        if feas <= tol:
            reason = "tolerance"
    plan = np.zeros((prob.m, prob.n))
    plan[np.ix_(rmask, cmask)] = X
    phi_full, psi_full = np.zeros(prob.m), np.zeros(prob.n)
    phi_full[rmask], psi_full[cmask] = phi, psi
    Xr = feasible_rounding(prob.f, prob.g, plan)
    robj = float(np.vdot(prob.C, Xr))
    dobj = float(prob.f @ phi_full + prob.g @ psi_full)
    return plan, phi_full, psi_full, dict(iterations=it, termination_reason=reason, final_relative_kkt=feas,
                                          rounded_objective=robj, duality_gap=abs(robj - dobj))
