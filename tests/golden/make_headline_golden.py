"""Reference-run fixtures at the HEADLINE configurations.

Runs the REFERENCE (`otsolve`, read-only from /root/reference/pkg/src) on the
benchmark instances and records its full trajectory:

    c2    m=n=4096  (64x64 grid) sq-Euclidean whitenoise seed 0, tol 1e-6
    c3    m=n=16384 (128x128 grid), tol 1e-4            (~20 s / iteration here)
    c4a   512 x 2048 analogue of C4 (L1 rect, sparse marginals) seed 0, tol 1e-4
    c4    C4 itself, 8192 x 32768 (~20 s / iteration here: the first iterations)
    c1s1, c1s2   C1 seeds 1 and 2 (1024^2, tol 1e-4) with traces
    c1p4, c2p4   C1 / C2 to tol 1e-8 (the converged objective)

    OPENBLAS_NUM_THREADS=1 OMP_NUM_THREADS=1 python tests/golden/make_headline_golden.py c2

Instances are built with the reference's own generators (synth_instance +
marginal_from_image, i.e. marginals normalised once) and the exact integer
cost of SURVEY F4; cost_fro_norm is pinned to the exact integer norm, which is
what the device problem uses (equal to np.linalg.norm(C) up to r = 64).

Every trace append is streamed to `_stream/<name>.jsonl` as it happens, so a
run that is stopped early still leaves a usable prefix (`--finalize` turns a
stream, complete or not, into the committed `headline_<name>.json`).  On
completion the script writes `headline_<name>.json` (report, objectives,
norms, the five trace lists, restart lengths) and `headline_<name>.npz` (the
returned plan's nonzeros, and the final duals).
"""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402

REF = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent
sys.path.insert(0, REF)
sys.path.insert(0, str(HERE.parents[1]))

import otsolve as ot  # noqa: E402

from paper_2407_19689_b200 import instances as inst  # noqa: E402

STREAM = HERE / "_stream"
TRACE_KEYS = ("etas", "step_bounds", "candidate_kkts", "omegas", "restart_kkts")

CASES = {
    "c2": dict(kind="sqeuclid", r=64, seed=0, tol=1e-6),
    "c3": dict(kind="sqeuclid", r=128, seed=0, tol=1e-4),
    "c4a": dict(kind="rect", src=(16, 32), dst=(32, 64), seed=0, tol=1e-4),
    "c4": dict(kind="rect", src=(64, 128), dst=(128, 256), seed=0, tol=1e-4),
    "c1p4": dict(kind="sqeuclid", r=32, seed=0, tol=1e-8),
    "c2p4": dict(kind="sqeuclid", r=64, seed=0, tol=1e-8),
    "c1s1": dict(kind="sqeuclid", r=32, seed=1, tol=1e-4),
    "c1s2": dict(kind="sqeuclid", r=32, seed=2, tol=1e-4),
}


def build(case):
    if case["kind"] == "sqeuclid":
        r = case["r"]
        src, dst = ot.synth_instance("whitenoise", r, case["seed"])
        prob = ot.OTProblem(ot.CostMatrix(inst.sqeuclid_grid_cost(r)), ot.marginal_from_image(src),
                            ot.marginal_from_image(dst))
        exact = inst.sqeuclid_fro_norm(r)
    else:
        s, d = case["src"], case["dst"]
        m, n = s[0] * s[1], d[0] * d[1]
        prob = ot.OTProblem(ot.CostMatrix(inst.rect_l1_cost(s, d)),
                            ot.Marginal(inst.sparse_weights(m, 2 * case["seed"])),
                            ot.Marginal(inst.sparse_weights(n, 2 * case["seed"] + 1)))
        exact = inst.rect_l1_fro_norm(s, d)
    prob.__dict__["cost_fro_norm"] = exact  # cached_property slot
    return prob


class _Stream(list):
    """A trace list that also appends every value to a JSONL file."""

    def __init__(self, key, fh, t0):
        super().__init__()
        self.key, self.fh, self.t0 = key, fh, t0

    def append(self, v):
        super().append(v)
        self.fh.write(json.dumps({"k": self.key, "v": float(v), "t": time.perf_counter() - self.t0}) + "\n")
        self.fh.flush()


class _Discard(list):
    """restart_points would hold an m x n copy per restart: not kept."""

    def append(self, v):
        pass


def _apply_A_longdouble(X):
    Xl = X.astype(np.longdouble)
    return Xl.sum(axis=1).astype(np.float64), Xl.sum(axis=0).astype(np.float64)


def _apply_A_reversed(X):
    Xr = X[::-1, ::-1]
    return Xr.sum(axis=1)[::-1].copy(), Xr.sum(axis=0)[::-1].copy()


def _apply_A_permuted(seed):
    """apply_A summed in a seeded random order: the rows of X are summed over a
    permuted column order and the columns over a permuted row order."""
    perms = {}

    def fn(X):
        m, n = X.shape
        if (m, n) not in perms:
            rng = np.random.default_rng(1000 + seed)
            perms[(m, n)] = (rng.permutation(n), rng.permutation(m))
        pc, pr = perms[(m, n)]
        return X[:, pc].sum(axis=1), X[pr, :].sum(axis=0)
    return fn


def _perturb(variant):
    """SURVEY A.3/A.8 self-drift envelope: the reference re-run with apply_A
    summed in long double ("ld"), in reversed order ("rev") or in a seeded
    random order ("rnd<k>"), patched at both import sites (pdhg_step /
    stepsize_bound and kkt_error)."""
    import otsolve.kkt as K
    import otsolve.pdhg as P
    if variant.startswith("rnd"):
        fn = _apply_A_permuted(int(variant[3:]))
    else:
        fn = {"ld": _apply_A_longdouble, "rev": _apply_A_reversed}[variant]
    P.apply_A = K.apply_A = fn


def run(name):
    base, _, variant = name.partition("_")
    case = dict(CASES[base])
    if variant:
        _perturb(variant)
        case["apply_A"] = variant
    prob = build(case)
    STREAM.mkdir(exist_ok=True)
    t0 = time.perf_counter()
    with open(STREAM / f"{name}.jsonl", "w") as fh:
        fh.write(json.dumps({"k": "meta", "case": case, "m": prob.m, "n": prob.n,
                             "cost_fro_norm": prob.cost_fro_norm, "marginal_norm": prob.marginal_norm,
                             "omp": os.environ.get("OMP_NUM_THREADS")}) + "\n")
        fh.flush()
        trace = ot.SolveTrace()
        for k in TRACE_KEYS:
            setattr(trace, k, _Stream(k, fh, t0))
        trace.restart_points = _Discard()
        # no wall-clock limit: C3 takes ~17 s per iteration here (SolverConfig's default
        # time_limit_s = 3600 would stop it after ~210 iterations)
        it, rep = ot.solve(prob, ot.SolverConfig(tol=case["tol"], deterministic=True, time_limit_s=1e9),
                           trace=trace)
        wall = time.perf_counter() - t0
        rows, cols = np.nonzero(it.X)
        np.savez_compressed(HERE / f"headline_{name}.npz", rows=rows.astype(np.int32),
                            cols=cols.astype(np.int32), vals=it.X[rows, cols], p=it.p, q=it.q)
        out = dict(case=case, m=prob.m, n=prob.n, cost_fro_norm=prob.cost_fro_norm,
                   marginal_norm=prob.marginal_norm, complete=rep.termination_reason == "tolerance",
                   iterations_recorded=rep.iterations, restart_lengths=list(rep.restart_lengths),
                   omp_num_threads=os.environ.get("OMP_NUM_THREADS"),
                   report=json.loads(rep.to_json()),
                   pre_rounding_objective=float(np.vdot(prob.C, it.X)),
                   dual_objective=float(prob.f @ it.p + prob.g @ it.q),
                   wall_s=wall, s_per_iteration=wall / max(1, rep.iterations),
                   trace={k: list(getattr(trace, k)) for k in TRACE_KEYS})
        (HERE / f"headline_{name}.json").write_text(json.dumps(out, indent=1, sort_keys=True))
        fh.write(json.dumps({"k": "done", "iterations": rep.iterations, "restarts": rep.restarts}) + "\n")
    print(name, rep.iterations, rep.restarts, rep.termination_reason, f"{wall:.0f}s")


def finalize(name):
    """Turn a (possibly partial) stream into headline_<name>.json."""
    lines = [json.loads(x) for x in (STREAM / f"{name}.jsonl").read_text().splitlines() if x.strip()]
    meta = lines[0]
    tr = {k: [] for k in TRACE_KEYS}
    t_last = 0.0
    restart_at = []  # total iterations at each restart (etas count when restart_kkts grows)
    for d in lines[1:]:
        if d["k"] in tr:
            tr[d["k"]].append(d["v"])
            t_last = d["t"]
            if d["k"] == "restart_kkts":
                restart_at.append(len(tr["etas"]))
    # the last streamed iteration's restart decision may still be in flight (the
    # restart is recorded after its candidate KKT): keep only iterations whose
    # successor has started, i.e. whose decisions are complete
    keep = max(0, min(len(tr["etas"]) - 1, len(tr["candidate_kkts"])))
    restart_at = [t for t in restart_at if t <= keep]
    nr = len(restart_at)
    tr = {"etas": tr["etas"][:keep], "step_bounds": tr["step_bounds"][:keep],
          "candidate_kkts": tr["candidate_kkts"][:keep], "omegas": tr["omegas"][:nr],
          "restart_kkts": tr["restart_kkts"][:nr]}
    lengths = [b - a for a, b in zip([0] + restart_at[:-1], restart_at)]
    done = any(d["k"] == "done" for d in lines)
    path = HERE / f"headline_{name}.json"
    if done and path.exists():
        print("complete fixture already written:", path)
        return
    out = dict(case=meta["case"], m=meta["m"], n=meta["n"], cost_fro_norm=meta["cost_fro_norm"],
               marginal_norm=meta["marginal_norm"], complete=False, omp_num_threads=meta["omp"],
               iterations_recorded=len(tr["etas"]), restarts_recorded=len(tr["omegas"]),
               s_per_iteration=t_last / max(1, len(tr["etas"])), restart_lengths=lengths, trace=tr)
    path.write_text(json.dumps(out, indent=1, sort_keys=True))
    print("partial fixture", path, len(tr["etas"]), "iterations")


if __name__ == "__main__":
    if "--finalize" in sys.argv:
        for nm in sys.argv[1:]:
            if nm != "--finalize":
                finalize(nm)
    else:
        for nm in sys.argv[1:]:
            run(nm)
