"""Pin the CPU oracle to the reference: bit-identical on the golden fixtures.

The fixtures were produced by the reference `otsolve` itself
(tests/golden/make_golden.py, single-threaded OpenBLAS).  The oracle must
reproduce every array and every report/trace scalar exactly; that is what
makes it a valid stand-in for the reference on the GPU box.
"""

import json
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import pdot_oracle as O
from paper_2407_19689_b200 import instances as inst

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def elements():
    return np.load(GOLD / "elements.npz")


@pytest.fixture(scope="module")
def solves():
    return np.load(GOLD / "solves.npz"), json.loads((GOLD / "solves.json").read_text())


def _cfg(**kw):
    base = dict(tol=1e-4, time_limit_s=3600.0, restart_mode="adaptive", beta=0.5,
                beta_sufficient=0.1, beta_necessary=0.9, beta_artificial=0.36, theta=0.5,
                eps_zero=1e-10, max_iters=1_000_000, deterministic=True, kkt_mode="relative",
                kkt_stride=1, eta0=None, omega0=1.0)
    base.update(kw)
    return SimpleNamespace(**base)


def raw_problem(C, f, g):
    return SimpleNamespace(C=C, f=f, g=g, m=C.shape[0], n=C.shape[1],
                           cost_fro_norm=float(np.linalg.norm(C)),
                           marginal_norm=float(np.linalg.norm(f) + np.linalg.norm(g)))


def test_element_functions_bit_identical(elements):
    E = elements
    for c in range(int(E["n_cases"][0])):
        k = lambda s: E[f"c{c}_{s}"]  # noqa: E731
        C, f, g, X, p, q = k("C"), k("f"), k("g"), k("X"), k("p"), k("q")
        tau, sigma, omega, scale_R = k("scal")
        Xn, pn, qn = O.primal_dual_step(C, f, g, X, p, q, tau, sigma)
        assert np.array_equal(Xn, k("Xn")) and np.array_equal(pn, k("pn")) and np.array_equal(qn, k("qn"))
        b = O.step_bound(X, p, q, Xn, pn, qn, omega)
        assert b == k("bound")[0]
        rows, cols = O.row_col_sums(X)
        assert np.array_equal(rows, k("rows")) and np.array_equal(cols, k("cols"))
        prob = raw_problem(C, f, g)
        rep = O.kkt_blocks(C, f, g, X, p, q, prob.cost_fro_norm, prob.marginal_norm, scale_R)
        assert [rep["gap"], rep["composite"], rep["relative_composite"]] == list(k("kkt"))
        assert np.array_equal(rep["dual_violation"], k("viol"))
        assert np.array_equal(O.feasible_rounding(f, g, X), k("Xr"))


def test_full_solves_bit_identical(solves):
    arrays, meta = solves
    for name, m in meta.items():
        # the fixture stores the reference's already-normalised marginals; use
        # them verbatim (re-normalising can move an entry by an ulp)
        prob = raw_problem(arrays[name + "_C"], arrays[name + "_f"], arrays[name + "_g"])
        init = None
        if name + "_X0" in arrays:
            init = SimpleNamespace(X=arrays[name + "_X0"], p=arrays[name + "_p0"], q=arrays[name + "_q0"])
        rec = O.new_record()
        (X, p, q), rep = O.oracle_solve(prob, _cfg(**m["config"]), initial=init, record=rec)
        ref = m["report"]
        for key in ("iterations", "restarts", "final_relative_kkt", "rounded_objective",
                    "duality_gap", "termination_reason", "restart_lengths", "restart_kkts", "solved"):
            assert rep[key] == ref[key], (name, key, rep[key], ref[key])
        assert rep["pre_rounding_objective"] == m["pre_rounding_objective"]
        assert np.array_equal(X, arrays[name + "_X"]), name
        assert np.array_equal(p, arrays[name + "_p"]) and np.array_equal(q, arrays[name + "_q"])
        for key in ("etas", "step_bounds", "candidate_kkts", "omegas", "restart_kkts"):
            assert rec[key] == m["trace"][key], (name, key)


def test_c1_seed0_report():
    """C1 (1024^2 whitenoise sq-Euclidean, tol 1e-4): 334 iterations / 21 restarts."""
    gold = json.loads((GOLD / "c1.json").read_text())["0"]
    prob = inst.sqeuclid_problem(32, 0)
    (X, p, q), rep = O.oracle_solve(prob, _cfg(tol=1e-4))
    for key in ("iterations", "restarts", "rounded_objective", "final_relative_kkt",
                "restart_lengths", "termination_reason"):
        assert rep[key] == gold["report"][key], key
    assert rep["pre_rounding_objective"] == gold["pre_rounding_objective"]


def test_instance_generators_match_reference():
    """grid_cost / synth images / grid_problem restated in instances.py are
    bit-identical to the reference's (fixtures from the reference itself)."""
    G = np.load(GOLD / "instances.npz")
    for kind in ("whitenoise", "shapes", "cauchy_like"):
        for norm in ("l1", "l2", "linf"):
            prob = inst.grid_problem(kind, 6, norm, 11)
            assert np.array_equal(prob.C, G[f"{kind}_{norm}_C"]), (kind, norm)
            assert np.array_equal(prob.f, G[f"{kind}_{norm}_f"]), (kind, norm)
            assert np.array_equal(prob.g, G[f"{kind}_{norm}_g"]), (kind, norm)


def test_sinkhorn_oracle_bit_identical():
    """oracle/sinkhorn_oracle.py reproduces the reference's sinkhorn_solve."""
    from oracle.sinkhorn_oracle import oracle_sinkhorn
    A = np.load(GOLD / "sinkhorn.npz")
    meta = json.loads((GOLD / "sinkhorn.json").read_text())
    for name, m in meta.items():
        prob = raw_problem(A[name + "_C"], A[name + "_f"], A[name + "_g"])
        plan, phi, psi, rep = oracle_sinkhorn(prob, m["penalty"], m["tol"])
        ref = m["report"]
        for key in ("iterations", "termination_reason", "final_relative_kkt", "rounded_objective", "duality_gap"):
            assert rep[key] == ref[key], (name, key, rep[key], ref[key])
        assert np.array_equal(plan, A[name + "_plan"]), name
        assert np.array_equal(phi, A[name + "_phi"]) and np.array_equal(psi, A[name + "_psi"]), name
