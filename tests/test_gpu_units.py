"""GPU parity of the unit entry points against the reference's golden vectors.

Golden arrays were produced by the reference itself (tests/golden/make_golden.py).
Tolerances:
  * X+ of pdhg_step, the dual-violation matrix and apply_At: BIT-IDENTICAL
    (element-wise arithmetic, no FMA contraction, same operation order);
  * everything that goes through a reduction (row/column sums, p+, q+, the
    step bound, KKT scalars, rounding): relative 1e-12 of the value's scale,
    because the GPU sums in a different (fixed, deterministic) order than
    numpy/OpenBLAS.
"""

from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def E():
    return np.load(GOLD / "elements.npz")


@pytest.fixture(scope="module")
def pd():
    import paper_2407_19689_b200 as pd
    return pd


def _raw(pd, C, f, g):
    from types import SimpleNamespace
    return SimpleNamespace(C=C, f=f, g=g, m=C.shape[0], n=C.shape[1],
                           cost_fro_norm=float(np.linalg.norm(C)),
                           marginal_norm=float(np.linalg.norm(f) + np.linalg.norm(g)))


def _close(a, b, rel=1e-12):
    a, b = np.asarray(a, float), np.asarray(b, float)
    scale = max(1.0, float(np.max(np.abs(b))) if b.size else 1.0)
    assert np.max(np.abs(a - b)) <= rel * scale, (np.max(np.abs(a - b)), scale)


def _cases(E):
    for c in range(int(E["n_cases"][0])):
        yield c, (lambda s, c=c: E[f"c{c}_{s}"])


def test_pdhg_step_golden(E, pd):
    for c, k in _cases(E):
        prob = _raw(pd, k("C"), k("f"), k("g"))
        tau, sigma, _, _ = k("scal")
        nxt = pd.pdhg_step(prob, pd.Iterate(k("X"), k("p"), k("q")), tau, sigma)
        assert np.array_equal(nxt.X, k("Xn")), f"case {c}: X+ not bit-identical"
        _close(nxt.p, k("pn"))
        _close(nxt.q, k("qn"))


def test_stepsize_bound_golden(E, pd):
    for c, k in _cases(E):
        it = pd.Iterate(k("X"), k("p"), k("q"))
        nx = pd.Iterate(k("Xn"), k("pn"), k("qn"))
        omega = k("scal")[2]
        b = pd.stepsize_bound(it, nx, omega)
        ref = k("bound")[0]
        assert b == pytest.approx(ref, rel=1e-11), c


def test_apply_A_golden(E, pd):
    for c, k in _cases(E):
        rows, cols = pd.apply_A(k("X"))
        _close(rows, k("rows"), 1e-13)
        _close(cols, k("cols"), 1e-13)


def test_kkt_error_golden(E, pd):
    for c, k in _cases(E):
        prob = _raw(pd, k("C"), k("f"), k("g"))
        scale_R = k("scal")[3]
        rep = pd.kkt_error(prob, pd.Iterate(k("X"), k("p"), k("q")), scale_R)
        gap, comp, rel = k("kkt")
        assert np.array_equal(rep.dual_violation, k("viol")), c
        _close(rep.primal_row, k("pr"), 1e-13)
        _close(rep.primal_col, k("pc"), 1e-13)
        assert rep.gap == pytest.approx(gap, rel=1e-11, abs=1e-13)
        assert rep.composite == pytest.approx(comp, rel=1e-12)
        assert rep.relative_composite == pytest.approx(rel, rel=1e-12)


def test_round_to_feasible_golden(E, pd):
    for c, k in _cases(E):
        prob = _raw(pd, k("C"), k("f"), k("g"))
        Xr = pd.round_to_feasible(prob, k("X"))
        _close(Xr, k("Xr"), 1e-12)
        np.testing.assert_allclose(Xr.sum(axis=1), k("f"), rtol=0, atol=1e-12)
        np.testing.assert_allclose(Xr.sum(axis=0), k("g"), rtol=0, atol=1e-12)
        assert np.all(Xr >= 0)


def test_apply_At_bit_identical(pd):
    rng = np.random.default_rng(0)
    for m, n in [(1, 1), (3, 5), (7, 2), (33, 65)]:
        p, q = rng.standard_normal(m), rng.standard_normal(n)
        assert np.array_equal(pd.apply_At(p, q), p[:, None] + q[None, :])


def test_step_matches_oracle_large(pd):
    """One step at a non-toy size: X+ bit-identical to the oracle, duals to 1e-12."""
    from oracle import pdot_oracle as O
    from paper_2407_19689_b200 import instances as inst
    prob = inst.sqeuclid_problem(16, 3)  # 256 x 256
    rng = np.random.default_rng(1)
    X = rng.random((256, 256)) * 1e-3
    X[rng.random(X.shape) < 0.4] = 0.0
    p, q = rng.standard_normal(256), rng.standard_normal(256)
    Xn, pn, qn = O.primal_dual_step(prob.C, prob.f, prob.g, X, p, q, 0.013, 0.7)
    nxt = pd.pdhg_step(prob, pd.Iterate(X, p, q), 0.013, 0.7)
    assert np.array_equal(nxt.X, Xn)
    _close(nxt.p, pn)
    _close(nxt.q, qn)


def test_running_average_bit_identical(pd):
    """A' = A + (X - A)/k in the fused kernel (Markstein division with a
    precomputed 1/k) is bit-identical to numpy's IEEE division, for many k;
    the dual average uses the trial duals as the solve loop does."""
    from oracle import pdot_oracle as O
    from paper_2407_19689_b200 import instances as inst
    from paper_2407_19689_b200.units import step_and_average
    prob = inst.sqeuclid_problem(16, 5)  # 256 x 256: full and edge tiles
    rng = np.random.default_rng(2)
    X = rng.random((256, 256)) * 1e-2
    X[rng.random(X.shape) < 0.5] = 0.0
    # averages with a wide spread of exponents, including exact zeros
    A = rng.random((256, 256)) * np.exp2(rng.integers(-60, 10, (256, 256)))
    A[rng.random(A.shape) < 0.2] = 0.0
    p, q = rng.standard_normal(256), rng.standard_normal(256)
    pa, qa = rng.standard_normal(256), rng.standard_normal(256)
    for k in (1, 2, 3, 7, 10, 49, 999, 123457):
        nxt, av = step_and_average(prob, pd.Iterate(X, p, q), pd.Iterate(A, pa, qa), 0.02, 0.3, k)
        Xn, _, _ = O.primal_dual_step(prob.C, prob.f, prob.g, X, p, q, 0.02, 0.3)
        assert np.array_equal(nxt.X, Xn)
        ref = A.copy()
        ref += (X - ref) / k           # pdhg.py:315 (average of the input iterate), IEEE division
        assert np.array_equal(av.X, ref), k
        rp = pa.copy()
        rp += (nxt.p - rp) / k         # pdhg.py:316 on the GPU's own p+
        rq = qa.copy()
        rq += (nxt.q - rq) / k
        assert np.array_equal(av.p, rp) and np.array_equal(av.q, rq), k
