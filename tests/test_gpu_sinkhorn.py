"""GPU log-domain Sinkhorn against the reference's own
runs (tests/golden/sinkhorn.*, produced by otsolve.sinkhorn_solve).

Tolerances: the GPU evaluates exp/log with CUDA's fp64 functions (<= 1 ulp,
different rounding than glibc) and sums in a fixed tree, so potentials agree
to ~1e-9 relative of their scale, the iteration count to +-1, and the
reported feasibility / objective to the run's tolerance."""

import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden"
A = np.load(GOLD / "sinkhorn.npz")
META = json.loads((GOLD / "sinkhorn.json").read_text())


def _raw(C, f, g):
    from types import SimpleNamespace
    return SimpleNamespace(C=C, f=f, g=g, m=C.shape[0], n=C.shape[1],
                           cost_fro_norm=float(np.linalg.norm(C)),
                           marginal_norm=float(np.linalg.norm(f) + np.linalg.norm(g)))


@pytest.mark.parametrize("name", sorted(META))
def test_sinkhorn_matches_reference(name):
    import paper_2407_19689_b200 as pd
    m = META[name]
    prob = _raw(A[name + "_C"], A[name + "_f"], A[name + "_g"])
    plan, pot, rep = pd.sinkhorn_solve(prob, pd.SinkhornConfig(penalty=m["penalty"], tol=m["tol"],
                                                               deterministic=True))
    ref = m["report"]
    print(name, rep.iterations, ref["iterations"], rep.final_relative_kkt, ref["final_relative_kkt"])
    assert rep.termination_reason == ref["termination_reason"] == "tolerance"
    assert abs(rep.iterations - ref["iterations"]) <= 1
    assert rep.final_relative_kkt <= m["tol"]
    scale = max(1.0, float(np.max(np.abs(A[name + "_phi"]))))
    if rep.iterations == ref["iterations"]:
        assert np.max(np.abs(pot.phi - A[name + "_phi"])) <= 1e-9 * scale
        assert np.max(np.abs(pot.psi - A[name + "_psi"])) <= 1e-9 * scale
        np.testing.assert_allclose(plan, A[name + "_plan"], rtol=1e-7, atol=1e-14)
    assert rep.rounded_objective == pytest.approx(ref["rounded_objective"], rel=1e-6, abs=1e-9)
    assert rep.method == "sinkhorn" and rep.restarts == 0


def test_sinkhorn_limits_and_errors():
    import paper_2407_19689_b200 as pd
    from paper_2407_19689_b200 import instances as inst
    prob = inst.grid_problem("whitenoise", 8, "l1", 1)
    _, _, rep = pd.sinkhorn_solve(prob, pd.SinkhornConfig(penalty=0.001, tol=1e-12, max_iters=7))
    assert rep.termination_reason == "iteration_limit" and rep.iterations == 7
    _, _, rep = pd.sinkhorn_solve(prob, pd.SinkhornConfig(penalty=0.001, tol=1e-14, time_limit_s=1e-4))
    assert rep.termination_reason == "time_limit"
    with pytest.raises(ValueError):
        pd.SinkhornConfig(penalty=0.0)


def test_sinkhorn_gap_below_pdot():
    """Acceptance-10 pattern (test_acceptance.py:287-310): the entropic gap
    exceeds PDOT's on the same instance."""
    import paper_2407_19689_b200 as pd
    from paper_2407_19689_b200 import instances as inst
    prob = inst.grid_problem("shapes", 16, "l1", 11)
    _, rep_p = pd.solve(prob, pd.SolverConfig(tol=1e-5))
    _, _, rep_s = pd.sinkhorn_solve(prob, pd.SinkhornConfig(penalty=0.01, tol=1e-4))
    assert rep_s.solved and rep_p.solved
    assert rep_s.duality_gap > rep_p.duality_gap
