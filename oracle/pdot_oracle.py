"""CPU oracle for the PDOT restarted-PDHG path — TEST INFRASTRUCTURE ONLY.

This module restates, in numpy, the algorithm of the reference package
``otsolve`` (reference tree ``/root/reference/pkg/src/otsolve``) so that the
CUDA path can be checked on the GPU box, where the reference tree does not
exist.  Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import it, and only as the
checker or the timed CPU baseline.  The product path
(``paper_2407_19689_b200``) never imports it: with the CUDA library missing the
product raises instead of falling back here.

Every numpy expression below is evaluated in the same order, with the same
temporaries and the same library calls (``ndarray.sum``, ``np.vdot``, ``@``,
``np.linalg.norm``) as the reference, so on the same machine and the same
OpenBLAS thread count it reproduces the reference bit for bit.  That claim is
pinned by ``tests/test_oracle_golden.py`` against fixtures that
``tests/golden/make_golden.py`` produced by running the reference itself.

Reference line citations are ``file:line`` relative to
``/root/reference/pkg/src/otsolve``.
"""

from __future__ import annotations

import math
import time

import numpy as np

GROWTH = 1.05  # pdhg.py:39 (_STEP_GROWTH)
HALVINGS = 80  # pdhg.py:40 (_MAX_HALVINGS)
ROUND_ZERO = 1e-14  # rounding.py:15 (ZERO_RESIDUAL_TOL)


# --------------------------------------------------------------------------
# operator.py
# --------------------------------------------------------------------------
def row_col_sums(X):
    """Constraint map A: (row sums, column sums).  operator.py:36-38."""
    return X.sum(axis=1), X.sum(axis=0)


def dual_broadcast(p, q):
    """Adjoint A^T: entry (i, j) = p_i + q_j.  operator.py:41-43."""
    return p[:, None] + q[None, :]


def stacked_norm(X, p, q):
    """Iterate.norm, kkt.py:36-42."""
    return float(np.sqrt(np.vdot(X, X) + np.vdot(p, p) + np.vdot(q, q)))


# --------------------------------------------------------------------------
# pdhg.py: one step and the step-size rule
# --------------------------------------------------------------------------
def primal_dual_step(C, f, g, X, p, q, tau, sigma):
    """pdhg.py:121-129.  Returns (X+, p+, q+)."""
    Xn = X - tau * (C - dual_broadcast(p, q))
    np.maximum(Xn, 0.0, out=Xn)
    rows, cols = row_col_sums(2.0 * Xn - X)
    return Xn, p + sigma * (f - rows), q + sigma * (g - cols)


def step_bound(X, p, q, Xn, pn, qn, omega, eps_zero=1e-10):
    """pdhg.py:132-149 (stepsize_bound)."""
    dX, dp, dq = Xn - X, pn - p, qn - q
    num = omega * float(np.vdot(dX, dX)) + (float(np.vdot(dp, dp)) + float(np.vdot(dq, dq))) / omega
    rows, cols = row_col_sums(dX)
    den = 2.0 * abs(float(dp @ rows + dq @ cols))
    return math.inf if den <= eps_zero else num / den


def eta_after_bound(bound, eta):
    """pdhg.py:152-171 (adaptive_stepsize) given an already computed bound."""
    if math.isinf(bound):
        return eta
    while eta > bound:
        eta *= 0.5
    return min(GROWTH * eta, bound)


def omega_update(dX, dpq, omega, theta=0.5, eps_zero=1e-10):
    """pdhg.py:174-186 (primal_weight_update)."""
    if omega <= 0:
        raise ValueError("omega_prev must be positive")
    if dX > eps_zero and dpq > eps_zero:
        return math.exp(theta * math.log(dpq / dX) + (1.0 - theta) * math.log(omega))
    return omega


def restart_fires(cfg, cand, start, prev, k, total):
    """pdhg.py:198-222 (should_restart)."""
    if cfg.restart_mode == "fixed":
        return cand <= cfg.beta * start
    if cand <= cfg.beta_sufficient * start:
        return True
    if cand <= cfg.beta_necessary * start and cand > prev:
        return True
    return k >= cfg.beta_artificial * total


# --------------------------------------------------------------------------
# kkt.py
# --------------------------------------------------------------------------
def kkt_blocks(C, f, g, X, p, q, fro_C, marg, scale_R=1.0):
    """kkt.py:56-94.  Returns a dict with the same fields as KKTReport."""
    if scale_R <= 0:
        raise ValueError("scale_R must be positive")
    rows, cols = row_col_sums(X)
    pr, pc = rows - f, cols - g
    viol = dual_broadcast(p, q) - C
    np.maximum(viol, 0.0, out=viol)
    pobj = float(np.vdot(C, X))
    dobj = float(f @ p + g @ q)
    gap = pobj - dobj
    psq = float(np.vdot(pr, pr) + np.vdot(pc, pc))
    dsq = float(np.vdot(viol, viol))
    comp = float(np.sqrt(psq + dsq + (gap / scale_R) ** 2))
    rel = np.sqrt(psq) / (1.0 + marg) + np.sqrt(dsq) / (1.0 + fro_C) + abs(gap) / (
        1.0 + abs(pobj) + abs(dobj)
    )
    return dict(primal_row=pr, primal_col=pc, dual_violation=viol, gap=gap,
                scale_R=float(scale_R), composite=comp, relative_composite=float(rel),
                primal_obj=pobj, dual_obj=dobj)


# --------------------------------------------------------------------------
# rounding.py
# --------------------------------------------------------------------------
def feasible_rounding(f, g, X):
    """rounding.py:18-40 (round_to_feasible)."""
    rs = X.sum(axis=1)
    with np.errstate(divide="ignore", invalid="ignore"):
        rscale = np.where(rs > 0, np.minimum(f / rs, 1.0), 1.0)
    Y = rscale[:, None] * X
    cs = Y.sum(axis=0)
    with np.errstate(divide="ignore", invalid="ignore"):
        cscale = np.where(cs > 0, np.minimum(g / cs, 1.0), 1.0)
    Y = Y * cscale[None, :]
    er = np.maximum(f - Y.sum(axis=1), 0.0)
    ec = np.maximum(g - Y.sum(axis=0), 0.0)
    tot = float(er.sum())
    if tot <= ROUND_ZERO:
        return Y
    return Y + np.outer(er, ec) / tot


# --------------------------------------------------------------------------
# pdhg.py:254-399 — the restarted loop, as an explicit state object
# --------------------------------------------------------------------------
class _Point:
    """(X, p, q) triple; Iterate in kkt.py:21-42."""

    __slots__ = ("X", "p", "q")

    def __init__(self, X, p, q):
        self.X, self.p, self.q = X, p, q

    def dup(self):
        return _Point(self.X.copy(), self.p.copy(), self.q.copy())

    def norm(self):
        return stacked_norm(self.X, self.p, self.q)


def oracle_solve(prob, cfg, initial=None, record=None, clock=time.perf_counter, on_iteration=None):
    """Restarted PDHG exactly as pdhg.py:254-399.

    ``prob`` is anything with ``C f g m n cost_fro_norm marginal_norm``;
    ``cfg`` anything with the SolverConfig fields (pdhg.py:43-59).
    ``initial`` is an object with ``X p q`` or None.  ``record`` is None or a
    dict that receives the SolveTrace lists (pdhg.py:106-118).

    Returns ``((X, p, q), report_dict)``; ``report_dict`` holds the
    SolveReport fields (reports.py:9-38) minus ``config_echo``, plus
    ``pre_rounding_objective`` (= <C, X> of the returned iterate).
    """
    C, f, g = prob.C, prob.f, prob.g
    m, n = prob.m, prob.n
    t0 = clock()
    fro_C, marg = prob.cost_fro_norm, prob.marginal_norm
    cur = _Point(np.zeros((m, n)), np.zeros(m), np.zeros(n)) if initial is None else \
        _Point(initial.X.copy(), initial.p.copy(), initial.q.copy())
    eta = cfg.eta0 if cfg.eta0 is not None else 1.0 / (2.0 * math.sqrt(m + n))  # pdhg.py:225-227
    omega = cfg.omega0
    adaptive = cfg.restart_mode == "adaptive"
    use_rel = cfg.kkt_mode == "relative"
    rec = record

    def score(rep):  # pdhg.py:275-276
        return rep["relative_composite"] if use_rel else rep["composite"]

    R = max(1.0, cur.norm())  # pdhg.py:278
    z_kkt = score(kkt_blocks(C, f, g, cur.X, cur.p, cur.q, fro_C, marg, R))
    anchor, avg = cur.dup(), cur.dup()  # pdhg.py:280-288
    kkts_at_restart = [z_kkt]
    lengths = []
    prev, best, best_kkt = z_kkt, cur.dup(), z_kkt
    outer = inner = total = 0
    reason = "tolerance" if z_kkt <= cfg.tol else None

    while reason is None:
        # loop-top limits, pdhg.py:299-306
        if total >= cfg.max_iters:
            reason, cur = "iteration_limit", best
            break
        if clock() - t0 > cfg.time_limit_s:
            reason, cur = "time_limit", best
            break
        # _accepted_step, pdhg.py:230-251
        if not adaptive:
            if rec is not None:
                rec["etas"].append(eta)
            nxt = _Point(*primal_dual_step(C, f, g, cur.X, cur.p, cur.q, eta / omega, eta * omega))
        else:
            for _ in range(HALVINGS):
                nxt = _Point(*primal_dual_step(C, f, g, cur.X, cur.p, cur.q, eta / omega, eta * omega))
                bnd = step_bound(cur.X, cur.p, cur.q, nxt.X, nxt.p, nxt.q, omega, cfg.eps_zero)
                if eta <= bnd:
                    if rec is not None:
                        rec["etas"].append(eta)
                        rec["step_bounds"].append(bnd)
                    if math.isfinite(bnd):
                        eta = min(GROWTH * eta, bnd)
                    break
                eta *= 0.5
            else:
                raise RuntimeError("step-size line search failed to find an admissible eta")
        cur = nxt
        total += 1
        inner += 1
        if on_iteration is not None:
            on_iteration(total)
        # running mean, pdhg.py:314-317
        avg.X += (cur.X - avg.X) / inner
        avg.p += (cur.p - avg.p) / inner
        avg.q += (cur.q - avg.q) / inner
        nrm = cur.norm()  # pdhg.py:319-322
        if not math.isfinite(nrm):
            raise RuntimeError("numerical failure: non-finite iterate")
        R = max(R, nrm)
        if rec is not None and rec.get("record_inner"):
            rec["inner_iterates"].append(cur.dup())
            rec["inner_averages"].append(avg.dup())
        if inner % cfg.kkt_stride != 0:
            continue
        k_cur = score(kkt_blocks(C, f, g, cur.X, cur.p, cur.q, fro_C, marg, R))
        k_avg = score(kkt_blocks(C, f, g, avg.X, avg.p, avg.q, fro_C, marg, R))
        cand, c_kkt = (cur, k_cur) if k_cur < k_avg else (avg, k_avg)  # tie -> average
        if rec is not None:
            rec["candidate_kkts"].append(c_kkt)
        if c_kkt < best_kkt:
            best, best_kkt = cand.dup(), c_kkt
        if c_kkt <= cfg.tol:
            cur, reason = cand.dup(), "tolerance"
            break
        if restart_fires(cfg, c_kkt, z_kkt, prev, inner, total):
            if adaptive:  # pdhg.py:352-362
                dX = float(np.linalg.norm(cand.X - anchor.X))
                dpq = float(np.sqrt(np.sum((cand.p - anchor.p) ** 2) + np.sum((cand.q - anchor.q) ** 2)))
                omega = omega_update(dX, dpq, omega, cfg.theta, cfg.eps_zero)
            cur = cand.dup()  # pdhg.py:363-376
            lengths.append(inner)
            kkts_at_restart.append(c_kkt)
            outer += 1
            inner = 0
            anchor, z_kkt, avg = cur.dup(), c_kkt, cur.dup()
            prev = c_kkt
            if rec is not None:
                rec["restart_points"].append(cur.dup())
                rec["restart_kkts"].append(c_kkt)
                rec["omegas"].append(omega)
        else:
            prev = c_kkt

    elapsed = clock() - t0  # pdhg.py:380-399
    fin = kkt_blocks(C, f, g, cur.X, cur.p, cur.q, fro_C, marg, R)
    Xr = feasible_rounding(f, g, cur.X)
    robj = float(np.vdot(C, Xr))
    dobj = float(f @ cur.p + g @ cur.q)
    report = dict(
        method="pdot",
        solved=reason == "tolerance",
        wall_time_s=0.0 if cfg.deterministic else float(elapsed),
        iterations=total,
        restarts=outer,
        final_relative_kkt=float(fin["relative_composite"]),
        rounded_objective=robj,
        duality_gap=abs(robj - dobj),
        termination_reason=reason,
        restart_lengths=list(lengths),
        restart_kkts=[float(v) for v in kkts_at_restart],
        pre_rounding_objective=float(np.vdot(C, cur.X)),
    )
    return (cur.X, cur.p, cur.q), report


def new_record(record_inner=False):
    """Empty SolveTrace-shaped dict (pdhg.py:106-118)."""
    return dict(record_inner=record_inner, etas=[], step_bounds=[], candidate_kkts=[],
                omegas=[], restart_points=[], restart_kkts=[], inner_iterates=[],
                inner_averages=[])
