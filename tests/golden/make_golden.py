"""Generate golden fixtures by running the REFERENCE (`otsolve`) itself.

Run here (the reference tree only exists in the build container):

    OPENBLAS_NUM_THREADS=1 OMP_NUM_THREADS=1 python tests/golden/make_golden.py

It imports `otsolve` read-only from /root/reference/pkg/src and writes small
`.npz` / `.json` fixtures next to this script.  The fixtures pin the oracle
(`oracle/pdot_oracle.py`, checked in `tests/test_oracle_golden.py`) and give
the GPU tests known answers that do not need the reference at run time.
"""

from __future__ import annotations

import json
import os
import sys
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


def ref_problem(C, f, g):
    """Reference problem from RAW weights: Marginal normalises them once."""
    return ot.OTProblem(ot.CostMatrix(C), ot.Marginal(f), ot.Marginal(g))


def ref_sqeuclid(r, seed):
    """The C1/C2/C3 family through the reference's own generators: whitenoise
    images from synth_instance, marginals from marginal_from_image (normalised
    once, instance.py:153-158), exact integer sq-Euclidean cost."""
    src, dst = ot.synth_instance("whitenoise", r, seed)
    return ot.OTProblem(ot.CostMatrix(inst.sqeuclid_grid_cost(r)), ot.marginal_from_image(src),
                        ot.marginal_from_image(dst))


def ref_rect(seed, src_shape, dst_shape):
    """The C4 family (builder-defined): raw sparse weights, normalised once."""
    m, n = src_shape[0] * src_shape[1], dst_shape[0] * dst_shape[1]
    return ref_problem(inst.rect_l1_cost(src_shape, dst_shape), inst.sparse_weights(m, 2 * seed),
                       inst.sparse_weights(n, 2 * seed + 1))


def random_problem(rng, m, n, margin=0.05):
    return ref_problem(rng.random((m, n)), rng.random(m) + margin, rng.random(n) + margin)


# ---------------------------------------------------------------------------
# element level: step, bound, kkt, rounding, apply_A on seeded inputs
# ---------------------------------------------------------------------------
ELEMENT_SHAPES = [(1, 1), (1, 5), (5, 1), (2, 3), (3, 5), (7, 7), (13, 9), (64, 96), (130, 70)]


def element_cases():
    out = {}
    rng = np.random.default_rng(20240717)
    for idx, (m, n) in enumerate(ELEMENT_SHAPES):
        prob = random_problem(rng, m, n)
        X = rng.random((m, n)) * rng.choice([0.01, 1.0])
        # zero some entries so the projection is exercised
        X[rng.random((m, n)) < 0.3] = 0.0
        p = rng.standard_normal(m)
        q = rng.standard_normal(n)
        tau, sigma, omega = float(rng.uniform(0.01, 2.0)), float(rng.uniform(0.01, 2.0)), float(
            rng.uniform(0.2, 5.0))
        it = ot.Iterate(X.copy(), p.copy(), q.copy())
        nxt = ot.pdhg_step(prob, it, tau, sigma)
        bound = ot.stepsize_bound(it, nxt, omega)
        scale_R = float(rng.uniform(1.0, 3.0))
        rep = ot.kkt_error(prob, it, scale_R)
        rows, cols = ot.apply_A(X)
        Xr = ot.round_to_feasible(prob, X)
        pre = f"c{idx}_"
        out.update({
            pre + "C": prob.C, pre + "f": prob.f, pre + "g": prob.g,
            pre + "X": X, pre + "p": p, pre + "q": q,
            pre + "scal": np.array([tau, sigma, omega, scale_R]),
            pre + "Xn": nxt.X, pre + "pn": nxt.p, pre + "qn": nxt.q,
            pre + "bound": np.array([bound]),
            pre + "rows": rows, pre + "cols": cols,
            pre + "kkt": np.array([rep.gap, rep.composite, rep.relative_composite]),
            pre + "pr": rep.primal_row, pre + "pc": rep.primal_col, pre + "viol": rep.dual_violation,
            pre + "Xr": Xr,
        })
    out["n_cases"] = np.array([len(ELEMENT_SHAPES)])
    return out


# ---------------------------------------------------------------------------
# trajectory level: full solves with SolveTrace
# ---------------------------------------------------------------------------
def solve_cases():
    cases = []
    rng = np.random.default_rng(7)
    cases.append(("rand5x4", random_problem(rng, 5, 4), dict(tol=1e-6), None))
    cases.append(("asym2x2", ref_problem([[0.0, 1.0], [1.0, 0.0]], [0.3, 0.7], [0.6, 0.4]),
                  dict(tol=1e-6), None))
    cases.append(("single", ref_problem([[0.0]], [1.0], [1.0]), dict(tol=1e-8), None))
    cases.append(("rand3x7_fixed", random_problem(rng, 3, 7),
                  dict(tol=1e-7, restart_mode="fixed", beta=0.5), None))
    cases.append(("rand6x6_stride3_abs", random_problem(rng, 6, 6),
                  dict(tol=1e-6, kkt_stride=3, kkt_mode="absolute"), None))
    cases.append(("rand4x4_limit", random_problem(rng, 4, 4), dict(tol=1e-14, max_iters=10), None))
    p = random_problem(rng, 5, 6)
    init = ot.Iterate(rng.random((5, 6)) * 0.05, rng.standard_normal(5) * 0.1,
                      rng.standard_normal(6) * 0.1)
    cases.append(("warm5x6", p, dict(tol=1e-6), init))
    for r, seed, tol in ((4, 0, 1e-6), (8, 1, 1e-4), (16, 0, 1e-4)):
        cases.append((f"sqeuc_r{r}_s{seed}", ref_sqeuclid(r, seed), dict(tol=tol), None))
    cases.append(("rect_l1_128x512", ref_rect(0, (8, 16), (16, 32)), dict(tol=1e-4), None))
    return cases


def instance_cases():
    """Reference instance generators on fixed seeds (pins instances.py)."""
    out = {}
    for kind in ("whitenoise", "shapes", "cauchy_like"):
        for norm in ("l1", "l2", "linf"):
            prob = ot.grid_problem(kind, 6, norm, seed=11)
            out[f"{kind}_{norm}_C"] = prob.C
            out[f"{kind}_{norm}_f"] = prob.f
            out[f"{kind}_{norm}_g"] = prob.g
    return out


def sinkhorn_cases():
    """Reference Sinkhorn runs (pins oracle/sinkhorn_oracle.py, checks the GPU)."""
    rng = np.random.default_rng(99)
    cases = [("rand5x4", random_problem(rng, 5, 4), 0.05, 1e-8),
             ("grid8_l1", ot.grid_problem("cauchy_like", 8, "l1", seed=2), 0.05, 1e-6),
             ("shapes16_l2", ot.grid_problem("shapes", 16, "l2", seed=11), 0.01, 1e-4)]
    f = inst.sparse_weights(128, 3)
    g = inst.sparse_weights(256, 4)
    cases.append(("rect_sparse", ref_problem(inst.rect_l1_cost((8, 16), (16, 16)) / 10.0, f, g), 0.05, 1e-6))
    arrays, meta = {}, {}
    for name, prob, pen, tol in cases:
        plan, pot, rep = ot.sinkhorn_solve(prob, ot.SinkhornConfig(penalty=pen, tol=tol, deterministic=True))
        arrays.update({name + "_C": prob.C, name + "_f": prob.f, name + "_g": prob.g, name + "_plan": plan,
                       name + "_phi": pot.phi, name + "_psi": pot.psi})
        meta[name] = dict(penalty=pen, tol=tol, report=json.loads(rep.to_json()))
        print("sinkhorn", name, rep.iterations, rep.termination_reason)
    np.savez_compressed(HERE / "sinkhorn.npz", **arrays)
    (HERE / "sinkhorn.json").write_text(json.dumps(meta, indent=1, sort_keys=True))


def main():
    sinkhorn_cases()
    np.savez_compressed(HERE / "instances.npz", **instance_cases())
    np.savez_compressed(HERE / "elements.npz", **element_cases())
    arrays = {}
    meta = {}
    for name, prob, cfgkw, init in solve_cases():
        cfg = ot.SolverConfig(deterministic=True, **cfgkw)
        trace = ot.SolveTrace()
        it, rep = ot.solve(prob, cfg, initial=init, trace=trace)
        arrays[name + "_C"] = prob.C
        arrays[name + "_f"] = prob.f
        arrays[name + "_g"] = prob.g
        arrays[name + "_X"] = it.X
        arrays[name + "_p"] = it.p
        arrays[name + "_q"] = it.q
        if init is not None:
            arrays[name + "_X0"] = init.X
            arrays[name + "_p0"] = init.p
            arrays[name + "_q0"] = init.q
        meta[name] = dict(
            config=cfgkw,
            report=json.loads(rep.to_json()),
            pre_rounding_objective=float(np.vdot(prob.C, it.X)),
            trace=dict(etas=trace.etas, step_bounds=trace.step_bounds,
                       candidate_kkts=trace.candidate_kkts, omegas=trace.omegas,
                       restart_kkts=trace.restart_kkts),
        )
        print(name, rep.iterations, rep.restarts, rep.termination_reason)
    np.savez_compressed(HERE / "solves.npz", **arrays)
    (HERE / "solves.json").write_text(json.dumps(meta, indent=1, sort_keys=True))

    # C1 (m = n = 1024, whitenoise, exact sq-Euclidean), tol 1e-4: report only
    c1 = {}
    for seed in (0,):
        prob = ref_sqeuclid(32, seed)
        trace = ot.SolveTrace()
        it, rep = ot.solve(prob, ot.SolverConfig(tol=1e-4, deterministic=True), trace=trace)
        c1[str(seed)] = dict(report=json.loads(rep.to_json()),
                             pre_rounding_objective=float(np.vdot(prob.C, it.X)),
                             dual_objective=float(prob.f @ it.p + prob.g @ it.q),
                             cost_fro_norm=prob.cost_fro_norm, marginal_norm=prob.marginal_norm,
                             trace=dict(etas=trace.etas, step_bounds=trace.step_bounds,
                                        candidate_kkts=trace.candidate_kkts, omegas=trace.omegas,
                                        restart_kkts=trace.restart_kkts))
        print("C1 seed", seed, rep.iterations, rep.restarts)
    (HERE / "c1.json").write_text(json.dumps(c1, indent=1, sort_keys=True))

    # objective parity at tight tolerance: 256^2 sq-Euclidean, tol 1e-8,
    # and C1 seeds 1-2 at tol 1e-4 (trajectory-sensitive; compared in the envelope)
    p4 = {}
    for r, seed, tol in ((16, 0, 1e-8), (16, 1, 1e-8), (16, 2, 1e-8), (32, 1, 1e-4), (32, 2, 1e-4)):
        prob = ref_sqeuclid(r, seed)
        it, rep = ot.solve(prob, ot.SolverConfig(tol=tol, deterministic=True))
        p4[f"r{r}_s{seed}_tol{tol:g}"] = dict(r=r, seed=seed, tol=tol, report=json.loads(rep.to_json()),
                                               pre_rounding_objective=float(np.vdot(prob.C, it.X)))
        print("P4", r, seed, tol, rep.iterations, rep.restarts, float(np.vdot(prob.C, it.X)))
    (HERE / "p4.json").write_text(json.dumps(p4, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
