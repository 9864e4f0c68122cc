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


def horizon(gpu_trace, gpu_lengths, ref_trace, ref_lengths, rtol=1e-10):
    """First iteration index (0-based) where the trajectories part, and why.

    Returns (h, reason, worst): all iterations < h agree within rtol (etas,
    step bounds, candidate KKTs, restart positions, omegas); ``worst`` is the
    largest relative difference seen inside the horizon."""
    ge, re_ = gpu_trace.etas, ref_trace["etas"]
    gb, rb = gpu_trace.step_bounds, ref_trace["step_bounds"]
    gc, rc = gpu_trace.candidate_kkts, ref_trace["candidate_kkts"]
    go, ro = gpu_trace.omegas, ref_trace["omegas"]
    gr, rr = restart_iterations(gpu_lengths), restart_iterations(ref_lengths)
    n = min(len(ge), len(re_))
    worst = 0.0
    ri = 0  # restarts passed so far
    for i in range(n):
        for nm, a, b in (("eta", ge, re_), ("bound", gb, rb), ("cand", gc, rc)):
            if i < len(a) and i < len(b):
                d = _rel(a[i], b[i])
                if d > rtol:
                    return i, f"{nm} differs by {d:.2e}", worst
                worst = max(worst, d)
        # restarts that fire after iteration i+1 (1-based count of iterations)
        g_here = [k for k, t in enumerate(gr) if t == i + 1]
        r_here = [k for k, t in enumerate(rr) if t == i + 1]
        if bool(g_here) != bool(r_here):
            return i, "restart decision differs", worst
        if g_here:
            if ri < len(go) and ri < len(ro):
                d = _rel(go[ri], ro[ri])
                if d > rtol:
                    return i, f"omega differs by {d:.2e}", worst
                worst = max(worst, d)
            ri += 1
    return n, "end of common trace", worst


def margins(events, config):
    """Per-iteration decision margins from the device event stream.

    Returns a list of dicts (one per accepted iteration) with the relative
    margins of: the candidate choice |kc - ka| / max, the acceptance
    (bound - eta) / eta, and the closest adaptive restart threshold."""
    out = []
    epoch = prev = None
    cur = {}
    k = 0
    total = 0
    for typ, ia, x, y, z in events:
        if typ == 1:  # START
            epoch = prev = x
        elif typ == 2:  # ACCEPT
            cur = {"accept": (y - x) / x if ia and math.isfinite(y) else math.inf}
            total += 1
            k += 1
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
            k = 0
    return out


def first_tight_decision(mg, below=1e-12):
    """Index of the first iteration whose smallest decision margin is < below."""
    for i, d in enumerate(mg):
        if min(d.values()) < below:
            return i, min(d, key=d.get), min(d.values())
    return None, None, None
