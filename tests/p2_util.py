"""Short-horizon trajectory parity between a GPU solve and a
reference-run trace.

The reference records, per accepted iteration, the step size eta and its
bound (pdhg.py:243-244) and the candidate KKT (pdhg.py:340); per restart the
candidate KKT and the updated primal weight omega (pdhg.py:374-376); and the
restart lengths in the report (pdhg.py:364).  `horizon` walks both traces in
iteration order and returns the first iteration at which any recorded value
differs by more than `rtol` relative, or a restart happens at a different
iteration -- the agreement horizon.  `margins` reports, from the GPU's own
device events, how close each discrete decision came to flipping (candidate
choice, acceptance, restart tests), so a divergence can be attributed to the
first decision whose margin is below the accumulated rounding difference.
"""

from __future__ import annotations

import math


def _rel(a, b):
    if a == b:
        return 0.0
    if math.isinf(a) or math.isinf(b):
        return math.inf
    return abs(a - b) / max(abs(a), abs(b), 1e-300)


def restart_iterations(lengths):
    out, tot = [], 0
    for k in lengths:
        tot += k
        out.append(tot)
    return out


def diffs(gpu_trace, gpu_lengths, ref_trace, ref_lengths):
    """Per-iteration comparison over the common prefix.

    Returns (d, split, why): d[i] = largest relative difference of iteration
    i's traced scalars (eta, step bound, candidate KKT, and omega at a restart);
    ``split`` = first iteration whose DISCRETE path differs -- a restart at a
    different iteration, or an eta off by more than 1e-3 relative (a different
    accept / reject sequence shows up as a factor-of-two eta) -- or the common
    length when the paths never split."""
    ge, re_ = gpu_trace.etas, ref_trace["etas"]
    gb, rb = gpu_trace.step_bounds, ref_trace["step_bounds"]
    gc, rc = gpu_trace.candidate_kkts, ref_trace["candidate_kkts"]
    go, ro = gpu_trace.omegas, ref_trace["omegas"]
    gr, rr = set(restart_iterations(gpu_lengths)), set(restart_iterations(ref_lengths))
    n = min(len(ge), len(re_))
    d = []
    ri = 0
    for i in range(n):
        di = 0.0
        for a, b in ((ge, re_), (gb, rb), (gc, rc)):
            if i < len(a) and i < len(b):
                di = max(di, _rel(a[i], b[i]))
        if _rel(ge[i], re_[i]) > 1e-3:
            return d, i, f"accept/reject path differs (eta rel diff {_rel(ge[i], re_[i]):.1e})"
        if ((i + 1) in gr) != ((i + 1) in rr):
            return d, i, "restart decision differs"
        if (i + 1) in gr:
            if ri < len(go) and ri < len(ro):
                di = max(di, _rel(go[ri], ro[ri]))
            ri += 1
        d.append(di)
    return d, n, "end of common trace"


def horizon(gpu_trace, gpu_lengths, ref_trace, ref_lengths, rtol=1e-10):
    """First iteration index (0-based) where the trajectories part by more
    than rtol, and why; (h, reason, worst) with ``worst`` the largest relative
    difference inside the horizon."""
    d, split, why = diffs(gpu_trace, gpu_lengths, ref_trace, ref_lengths)
    worst = 0.0
    for i, di in enumerate(d):
        if di > rtol:
            return i, f"a traced scalar differs by {di:.2e}", worst
        worst = max(worst, di)
    return split, why, worst


def decision_horizon(gpu_trace, gpu_lengths, ref_trace, ref_lengths):
    """(split, why, drift): the first iteration whose discrete path differs
    and the largest relative scalar difference accumulated before it."""
    d, split, why = diffs(gpu_trace, gpu_lengths, ref_trace, ref_lengths)
    return split, why, max(d) if d else 0.0


def growth(d, points=(10, 25, 50, 100, 200, 400, 800, 1600, 3200)):
    """Running maximum of the per-iteration difference at a few checkpoints."""
    out, run = {}, 0.0
    for i, di in enumerate(d):
        run = max(run, di)
        if i + 1 in points:
            out[i + 1] = run
    return out


def margins(events, config):
    """Per-iteration decision margins from the device event stream.

    Returns a list of dicts (one per accepted iteration) with the relative
    margins of: the candidate choice |kc - ka| / max, the acceptance
    (bound - eta) / eta, and the closest adaptive restart threshold."""
    out = []
    epoch = prev = None
    cur = {}
    for typ, ia, x, y, z in events:
        if typ == 1:  # START
            epoch = prev = x
        elif typ == 2:  # ACCEPT
            cur = {"accept": (y - x) / x if ia and math.isfinite(y) else math.inf}
        elif typ == 3:  # CAND: x cand, y current, z average
            cur["cand_choice"] = abs(y - z) / max(abs(y), abs(z), 1e-300)
            th = [abs(x - config.beta_sufficient * epoch) / x, abs(x - config.beta_necessary * epoch) / x]
            if x <= config.beta_necessary * epoch:
                th.append(abs(x - prev) / x)
            cur["restart"] = min(th)
            cur["tol"] = abs(x - config.tol) / config.tol
            prev = x
            out.append(cur)
        elif typ == 4:  # RESTART
            epoch = prev = x
    return out


def first_tight_decision(mg, below=1e-12):
    """Index of the first iteration whose smallest decision margin is < below.
    An exact candidate tie (current == average bit for bit, e.g. k = 1, where
    the average IS the iterate) is resolved identically by both sides (tie ->
    average) and is not a tight decision."""
    for i, d in enumerate(mg):
        d = {k: v for k, v in d.items() if not (k == "cand_choice" and v == 0.0)}
        if d and min(d.values()) < below:
            return i, min(d, key=d.get), min(d.values())
    return None, None, None
