"""The reference's own hot-path tests, re-targeted at the GPU path.

Each test restates a case of /root/reference/pkg/tests (file:line in the
docstring) with the reference's tolerance, calling paper_2407_19689_b200
instead of otsolve.  Independent oracles: dense PDHG on the materialised
constraint matrix (test_pdhg.py:55-66), hand-evaluated values, and HiGHS
(scipy.optimize.linprog) for the exact optimum of small instances in place
of the reference's spanning-tree enumeration (acceptance 6).
"""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pd():
    import paper_2407_19689_b200 as pd
    return pd


def make_problem(pd, C, f, g):
    return pd.make_problem(np.asarray(C, float), np.asarray(f, float), np.asarray(g, float))


def random_problem(pd, rng, m, n, margin=0.05):  # _helpers.py:12-17
    return make_problem(pd, rng.random((m, n)), rng.random(m) + margin, rng.random(n) + margin)


def two_by_two_optimal(pd):  # _helpers.py:24-28
    prob = make_problem(pd, [[0.0, 1.0], [1.0, 0.0]], [0.5, 0.5], [0.5, 0.5])
    return prob, pd.Iterate(np.diag([0.5, 0.5]), np.zeros(2), np.zeros(2))


def materialize_A(m, n):  # operator.py:46-56 (test oracle)
    return np.vstack([np.kron(np.eye(m), np.ones((1, n))), np.kron(np.ones((1, m)), np.eye(n))])


# --------------------------------------------------------------------------- test_pdhg.py
class TestPdhgStep:
    def test_fixed_point_at_optimum(self, pd):  # test_pdhg.py:70-75
        prob, it = two_by_two_optimal(pd)
        nxt = pd.pdhg_step(prob, it, tau=0.2, sigma=0.2)
        np.testing.assert_allclose(nxt.X, it.X, rtol=0, atol=1e-14)
        np.testing.assert_allclose(nxt.p, it.p, rtol=0, atol=1e-14)
        np.testing.assert_allclose(nxt.q, it.q, rtol=0, atol=1e-14)

    def test_from_zero_start(self, pd):  # test_pdhg.py:77-82
        prob, _ = two_by_two_optimal(pd)
        nxt = pd.pdhg_step(prob, pd.Iterate.zeros(2, 2), tau=0.1, sigma=0.1)
        np.testing.assert_array_equal(nxt.X, np.zeros((2, 2)))
        np.testing.assert_allclose(nxt.p, 0.1 * prob.f, rtol=0, atol=1e-16)
        np.testing.assert_allclose(nxt.q, 0.1 * prob.g, rtol=0, atol=1e-16)

    def test_matches_dense_vectorized_pdhg(self, pd):  # test_pdhg.py:84-100 + acceptance 4
        rng = np.random.default_rng(4)
        for _ in range(20):
            m, n = int(rng.integers(1, 6)), int(rng.integers(1, 6))
            prob = random_problem(pd, rng, m, n)
            A = materialize_A(m, n)
            c, b = prob.C.ravel(), np.concatenate([prob.f, prob.g])
            eta = pd.default_stepsize(prob)
            it = pd.Iterate(rng.random((m, n)), rng.standard_normal(m), rng.standard_normal(n))
            x, y = it.X.ravel().copy(), np.concatenate([it.p, it.q])
            for _ in range(50):
                x_new = np.maximum(x - eta * (c - A.T @ y), 0.0)
                y = y + eta * (b - A @ (2.0 * x_new - x))
                x = x_new
                it = pd.pdhg_step(prob, it, eta, eta)
                assert np.max(np.abs(it.X.ravel() - x)) <= 1e-10
                assert np.max(np.abs(np.concatenate([it.p, it.q]) - y)) <= 1e-10


class TestStepSize:  # test_pdhg.py:103-132
    def test_zero_displacement_keeps_eta(self, pd):
        it = pd.Iterate.zeros(2, 2)
        assert pd.adaptive_stepsize(it, it.copy(), omega=1.0, eta_current=0.7) == 0.7

    def test_hand_evaluated_bound(self, pd):
        it = pd.Iterate.zeros(2, 2)
        nxt = pd.Iterate(np.array([[1.0, 0.0], [0.0, 0.0]]), np.array([1.0, 0.0]), np.zeros(2))
        assert pd.stepsize_bound(it, nxt, omega=1.0) == pytest.approx(1.0, abs=1e-15)
        assert pd.adaptive_stepsize(it, nxt, omega=1.0, eta_current=4.0) == pytest.approx(1.0, abs=1e-15)
        assert pd.adaptive_stepsize(it, nxt, omega=1.0, eta_current=0.1) == pytest.approx(0.105)
        assert pd.adaptive_stepsize(it, nxt, omega=1.0, eta_current=0.99) == pytest.approx(1.0)


class TestRestartCandidate:  # test_pdhg.py:147-163
    def test_choice_and_tie(self, pd):
        prob, opt = two_by_two_optimal(pd)
        worse = pd.Iterate.zeros(2, 2)
        assert pd.restart_candidate(opt, worse, prob, scale_R=1.0) is opt
        assert pd.restart_candidate(worse, opt, prob, scale_R=1.0) is opt
        assert pd.restart_candidate(opt, opt.copy(), prob, scale_R=1.0) is not opt


class TestSolve:  # test_pdhg.py:187-285
    def test_forced_single_cell(self, pd):
        prob = make_problem(pd, [[0.0]], [1.0], [1.0])
        _, report = pd.solve(prob, pd.SolverConfig(tol=1e-8))
        assert report.solved
        assert report.rounded_objective == 0.0
        assert report.duality_gap <= 1e-7

    def test_asymmetric_two_by_two(self, pd):
        prob = make_problem(pd, [[0.0, 1.0], [1.0, 0.0]], [0.3, 0.7], [0.6, 0.4])
        it, report = pd.solve(prob, pd.SolverConfig(tol=1e-6))
        assert report.solved
        assert report.rounded_objective == pytest.approx(0.3, abs=1e-4)
        assert np.all(np.isfinite(it.X))

    def test_warm_start_at_optimum(self, pd):
        prob, opt = two_by_two_optimal(pd)
        _, report = pd.solve(prob, pd.SolverConfig(tol=1e-6), initial=opt)
        assert report.solved and report.iterations == 0

    def test_fixed_beta_restart_decay(self, pd):
        rng = np.random.default_rng(5)
        prob = random_problem(pd, rng, 4, 4)
        _, report = pd.solve(prob, pd.SolverConfig(restart_mode=pd.FIXED_BETA, beta=0.5, tol=1e-7))
        assert report.solved and report.restarts >= 3
        kkts = report.restart_kkts
        for prev, nxt in zip(kkts, kkts[1:]):
            assert nxt <= 0.5 * prev

    def test_accepted_steps_satisfy_bound(self, pd):
        rng = np.random.default_rng(6)
        prob = random_problem(pd, rng, 3, 5)
        trace = pd.SolveTrace()
        _, report = pd.solve(prob, pd.SolverConfig(tol=1e-6), trace=trace)
        assert report.solved
        assert len(trace.etas) == report.iterations
        for eta, bound in zip(trace.etas, trace.step_bounds):
            assert eta <= bound

    def test_running_average_recursion(self, pd):
        rng = np.random.default_rng(8)
        prob = random_problem(pd, rng, 3, 3)
        trace = pd.SolveTrace(record_inner=True)
        cfg = pd.SolverConfig(restart_mode=pd.FIXED_BETA, beta=1e-9, tol=1e-16, max_iters=25)
        pd.solve(prob, cfg, trace=trace)
        assert len(trace.inner_iterates) == 25
        mean_X = np.mean([z.X for z in trace.inner_iterates], axis=0)
        np.testing.assert_allclose(trace.inner_averages[-1].X, mean_X, rtol=0, atol=1e-13)
        mean_p = np.mean([z.p for z in trace.inner_iterates], axis=0)
        np.testing.assert_allclose(trace.inner_averages[-1].p, mean_p, rtol=0, atol=1e-13)

    def test_iteration_limit(self, pd):
        rng = np.random.default_rng(9)
        prob = random_problem(pd, rng, 4, 4)
        _, report = pd.solve(prob, pd.SolverConfig(tol=1e-14, max_iters=10))
        assert not report.solved
        assert report.termination_reason == "iteration_limit"
        assert report.iterations == 10

    def test_time_limit(self, pd):
        rng = np.random.default_rng(10)
        prob = random_problem(pd, rng, 8, 8)
        _, report = pd.solve(prob, pd.SolverConfig(tol=1e-16, time_limit_s=1e-4, max_iters=10**9))
        assert not report.solved
        assert report.termination_reason == "time_limit"

    def test_time_limit_mid_solve(self, pd):
        """The device deadline stops a long run close to the limit."""
        prob = pd.DeviceProblem.sqeuclid_grid(64, 0)
        # 0.2 s: C2 at ~24k iterations/s reaches even rel-KKT 1e-16 after ~10k iterations
        _, report = pd.solve(prob, pd.SolverConfig(tol=1e-16, time_limit_s=0.2, max_iters=10**9))
        assert report.termination_reason == "time_limit"
        assert report.iterations > 100
        assert report.wall_time_s < 0.2 + 0.5  # the host notices the device deadline at its next poll

    def test_iterates_stay_finite(self, pd):
        rng = np.random.default_rng(12)
        prob = random_problem(pd, rng, 5, 3)
        it, report = pd.solve(prob, pd.SolverConfig(tol=1e-6))
        assert math.isfinite(it.norm())
        assert report.final_relative_kkt <= 1e-6

    def test_whitenoise_grid_self_certifies(self, pd):
        from paper_2407_19689_b200 import instances as inst
        prob = inst.grid_problem("whitenoise", 16, "l2", seed=11)
        _, report = pd.solve(prob, pd.SolverConfig(tol=1e-5))
        assert report.solved
        assert report.final_relative_kkt <= 1e-4
        assert report.duality_gap <= 1e-3 * (1.0 + abs(report.rounded_objective))

    def test_report_round_trip(self, pd):
        prob = make_problem(pd, [[0.0, 1.0], [1.0, 0.0]], [0.3, 0.7], [0.6, 0.4])
        _, report = pd.solve(prob, pd.SolverConfig(tol=1e-5))
        assert pd.SolveReport.from_json(report.to_json()) == report

    def test_restart_points_recorded(self, pd):
        rng = np.random.default_rng(13)
        prob = random_problem(pd, rng, 4, 5)
        trace = pd.SolveTrace()
        _, report = pd.solve(prob, pd.SolverConfig(tol=1e-6), trace=trace)
        assert len(trace.restart_points) == report.restarts == len(trace.omegas)
        assert trace.restart_kkts == report.restart_kkts[1:]


# --------------------------------------------------------------------------- test_kkt.py
class TestKKT:
    def test_optimal_point_vanishes(self, pd):  # test_kkt.py:10-15
        prob, it = two_by_two_optimal(pd)
        rep = pd.kkt_error(prob, it, scale_R=1.0)
        assert rep.composite == 0.0 and rep.relative_composite == 0.0 and rep.gap == 0.0

    def test_hand_evaluated_display(self, pd):  # test_kkt.py:17-26
        prob, it = two_by_two_optimal(pd)
        it.p = np.array([1.0, 0.0])
        rep = pd.kkt_error(prob, it, scale_R=1.0)
        np.testing.assert_array_equal(rep.primal_row, [0.0, 0.0])
        np.testing.assert_array_equal(rep.primal_col, [0.0, 0.0])
        np.testing.assert_array_equal(rep.dual_violation, [[1.0, 0.0], [0.0, 0.0]])
        assert rep.gap == -0.5
        assert rep.composite == pytest.approx(np.sqrt(1.25), abs=1e-15)

    def test_zero_iterate_pure_primal(self, pd):  # test_kkt.py:28-33
        prob, _ = two_by_two_optimal(pd)
        rep = pd.kkt_error(prob, pd.Iterate.zeros(2, 2), scale_R=1.0)
        assert rep.composite == pytest.approx(float(np.sqrt(np.sum(prob.f**2) + np.sum(prob.g**2))), abs=1e-15)

    def test_scale_R(self, pd):  # test_kkt.py:35-47
        prob, it = two_by_two_optimal(pd)
        it.p = np.array([1.0, 1.0])
        r1 = pd.kkt_error(prob, it, scale_R=1.0)
        r2 = pd.kkt_error(prob, it, scale_R=2.0)
        assert r1.gap == r2.gap == -1.0
        assert r1.composite > r2.composite
        with pytest.raises(ValueError):
            pd.kkt_error(prob, it, scale_R=0.0)

    def test_relative_composite_formula(self, pd):  # test_kkt.py:58-75
        rng = np.random.default_rng(3)
        prob = make_problem(pd, rng.random((3, 4)), rng.random(3) + 0.1, rng.random(4) + 0.1)
        it = pd.Iterate(rng.random((3, 4)), rng.standard_normal(3), rng.standard_normal(4))
        rep = pd.kkt_error(prob, it, scale_R=2.5)
        pr = it.X.sum(axis=1) - prob.f
        pc = it.X.sum(axis=0) - prob.g
        dv = np.maximum(it.p[:, None] + it.q[None, :] - prob.C, 0.0)
        pobj, dobj = float(np.vdot(prob.C, it.X)), float(prob.f @ it.p + prob.g @ it.q)
        expected = (np.sqrt(np.sum(pr**2) + np.sum(pc**2)) / (1.0 + np.linalg.norm(prob.f) + np.linalg.norm(prob.g))
                    + np.linalg.norm(dv) / (1.0 + np.linalg.norm(prob.C))
                    + abs(pobj - dobj) / (1.0 + abs(pobj) + abs(dobj)))
        assert rep.relative_composite == pytest.approx(expected, rel=1e-14)

    def test_duality_gap(self, pd):  # test_kkt.py:105-120
        prob, it = two_by_two_optimal(pd)
        assert pd.duality_gap(prob, it) == 0.0
        it.p = np.array([1.0, 1.0])
        assert pd.duality_gap(prob, it) == 1.0
        rng = np.random.default_rng(9)
        prob = make_problem(pd, rng.random((3, 4)), rng.random(3) + 0.1, rng.random(4) + 0.1)
        plan = np.outer(prob.f, prob.g)
        assert pd.duality_gap(prob, pd.Iterate(plan, np.zeros(3), np.zeros(4))) == pytest.approx(
            float(np.vdot(prob.C, plan)), rel=1e-14)


# --------------------------------------------------------------------------- test_operator.py + acceptance 1
class TestOperator:
    def test_direct(self, pd):  # test_operator.py:14-37
        rows, cols = pd.apply_A(np.array([[1.0, 2.0], [3.0, 4.0]]))
        assert rows.tolist() == [3.0, 7.0] and cols.tolist() == [4.0, 6.0]
        out = pd.apply_At(np.array([1.0, 2.0]), np.array([10.0, 20.0]))
        assert out.tolist() == [[11.0, 21.0], [12.0, 22.0]]
        rows, cols = pd.apply_A(pd.apply_At(np.array([1.0, 0.0]), np.array([0.0, 0.0])))
        assert rows.tolist() == [2.0, 0.0] and cols.tolist() == [1.0, 1.0]

    def test_matches_materialized(self, pd):  # acceptance 1 (test_acceptance.py:120-137)
        rng = np.random.default_rng(1)
        for m in range(1, 7):
            for n in range(1, 7):
                A = materialize_A(m, n)
                for _ in range(5):
                    X = rng.standard_normal((m, n))
                    rows, cols = pd.apply_A(X)
                    assert np.max(np.abs(A @ X.ravel() - np.concatenate([rows, cols]))) <= 1e-14
                    p, q = rng.standard_normal(m), rng.standard_normal(n)
                    ref = (A.T @ np.concatenate([p, q])).reshape(m, n)
                    assert np.max(np.abs(ref - pd.apply_At(p, q))) <= 1e-14


# --------------------------------------------------------------------------- test_rounding.py + acceptance 5
class TestRounding:
    def test_hand_cases(self, pd):  # test_rounding.py:15-38
        prob = make_problem(pd, [[0.0, 1.0], [1.0, 0.0]], [0.5, 0.5], [0.5, 0.5])
        np.testing.assert_allclose(pd.round_to_feasible(prob, np.diag([0.5, 0.5])), np.diag([0.5, 0.5]),
                                   rtol=0, atol=1e-15)
        np.testing.assert_allclose(pd.round_to_feasible(prob, np.diag([0.6, 0.6])), np.diag([0.5, 0.5]),
                                   rtol=0, atol=1e-15)
        np.testing.assert_allclose(pd.round_to_feasible(prob, np.diag([0.4, 0.4])),
                                   [[0.45, 0.05], [0.05, 0.45]], rtol=0, atol=1e-15)

    def test_random_feasible_and_bounded(self, pd):  # acceptance 5 (test_acceptance.py:203-219)
        rng = np.random.default_rng(5)
        for _ in range(200):
            m, n = int(rng.integers(1, 8)), int(rng.integers(1, 8))
            prob = random_problem(pd, rng, m, n)
            X = rng.random((m, n)) * float(rng.choice([0.05, 1.0, 5.0]))
            Xf = pd.round_to_feasible(prob, X)
            assert np.all(Xf >= 0)
            assert np.max(np.abs(Xf.sum(axis=1) - prob.f)) <= 1e-12
            assert np.max(np.abs(Xf.sum(axis=0) - prob.g)) <= 1e-12
            lhs = float(np.abs(Xf - X).sum())
            rhs = 2.0 * (float(np.abs(prob.f - X.sum(axis=1)).sum()) + float(np.abs(prob.g - X.sum(axis=0)).sum()))
            assert lhs <= rhs + 1e-12 * (1.0 + rhs)  # Lemma 2, rounding.py:43-50

    def test_idempotent(self, pd):  # test_rounding.py:84-90
        rng = np.random.default_rng(77)
        for _ in range(20):
            prob = random_problem(pd, rng, 4, 3)
            Xf = pd.round_to_feasible(prob, rng.random((4, 3)))
            np.testing.assert_allclose(pd.round_to_feasible(prob, Xf), Xf, rtol=0, atol=1e-14)


# --------------------------------------------------------------------------- acceptance 6 / 7 / 12
def test_acceptance6_exact_recovery(pd):
    """50 small instances (m+n <= 9) solved to 1e-6 match the exact LP optimum
    within 1e-4(1+|opt|) (test_acceptance.py:222-242); exact optimum by HiGHS."""
    from scipy.optimize import linprog
    rng = np.random.default_rng(101)
    worst = 0.0
    for _ in range(50):
        while True:
            m, n = int(rng.integers(2, 6)), int(rng.integers(2, 6))
            if m + n <= 9:
                break
        prob = random_problem(pd, rng, m, n)
        res = linprog(prob.C.ravel(), A_eq=materialize_A(m, n), b_eq=np.concatenate([prob.f, prob.g]),
                      bounds=(0, None), method="highs")
        assert res.status == 0
        _, report = pd.solve(prob, pd.SolverConfig(tol=1e-6))
        assert report.solved
        err = abs(report.rounded_objective - res.fun) / (1.0 + abs(res.fun))
        worst = max(worst, err)
        assert err <= 1e-4
    print(f"acceptance 6: worst scaled error {worst:.2e}")


@pytest.mark.parametrize("cls", ["shapes", "cauchy_like"])
@pytest.mark.parametrize("norm", ["l1", "l2", "linf"])
def test_acceptance7_self_certified_scale(pd, cls, norm):
    """Six 256x256 instances from 16x16 grids solve to rel-KKT <= 1e-4 with the
    post-rounding gap below 1e-3(1+|obj|) (test_acceptance.py:52-68, 245-257)."""
    from paper_2407_19689_b200 import instances as inst
    prob = inst.grid_problem(cls, 16, norm, seed=11)
    _, report = pd.solve(prob, pd.SolverConfig(tol=1e-5, max_iters=200_000))
    assert report.solved
    assert report.final_relative_kkt <= 1e-4
    assert report.duality_gap <= 1e-3 * (1.0 + abs(report.rounded_objective))


def test_acceptance12_deterministic_reports(pd):
    """Two deterministic solves give byte-identical JSON (test_acceptance.py:335-351)."""
    from paper_2407_19689_b200 import instances as inst
    prob = inst.grid_problem("cauchy_like", 4, "l2", seed=3)
    payloads = [pd.solve(prob, pd.SolverConfig(tol=1e-6, deterministic=True))[1].to_json() for _ in range(2)]
    assert payloads[0] == payloads[1]


def test_nonfinite_raises(pd):
    """A non-finite iterate raises the reference's RuntimeError (pdhg.py:319-321)."""
    prob = make_problem(pd, [[0.0, 1.0], [1.0, 0.0]], [0.5, 0.5], [0.5, 0.5])
    bad = pd.Iterate(np.array([[np.inf, 0.0], [0.0, 0.5]]), np.zeros(2), np.zeros(2))
    with pytest.raises(RuntimeError):
        pd.solve(prob, pd.SolverConfig(tol=1e-6, restart_mode=pd.FIXED_BETA), initial=bad)


def test_acceptance12_cli_byte_identical(tmp_path):
    """`gen` + two `solve --deterministic` runs write byte-identical reports
    (test_acceptance.py:335-351, through this package's CLI)."""
    from paper_2407_19689_b200.cli import main as cli_main
    inst_file = tmp_path / "inst.txt"
    assert cli_main(["gen", "--class", "cauchy_like", "--resolution", "4", "--norm", "l2", "--seed", "3",
                     "--out", str(inst_file)]) == 0
    payloads = []
    for name in ("r1.json", "r2.json"):
        out = tmp_path / name
        assert cli_main(["solve", "--instance", str(inst_file), "--method", "pdot", "--tol", "1e-6",
                         "--deterministic", "--out", str(out)]) == 0
        payloads.append(out.read_bytes())
    assert payloads[0] == payloads[1]
