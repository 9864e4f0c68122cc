"""Host-side logic that needs no GPU: configuration validation, the scalar
rules, records.  Cases mirror the reference tests (test_pdhg.py:103-156,
257-299) so the drop-in behaves the same at its Python boundary."""

import math

import numpy as np
import pytest

import paper_2407_19689_b200 as pd
from paper_2407_19689_b200.config import eta_from_bound


class TestConfigValidation:  # test_pdhg.py:288-299, pdhg.py:61-75
    def test_rejects_bad_beta(self):
        with pytest.raises(ValueError):
            pd.SolverConfig(beta=1.5)

    def test_rejects_bad_mode(self):
        with pytest.raises(ValueError):
            pd.SolverConfig(restart_mode="sometimes")

    def test_rejects_bad_stride(self):
        with pytest.raises(ValueError):
            pd.SolverConfig(kkt_stride=0)

    @pytest.mark.parametrize("kw", [dict(tol=0), dict(time_limit_s=-1), dict(max_iters=0),
                                    dict(beta_sufficient=0.95), dict(kkt_mode="l2"), dict(omega0=0),
                                    dict(eta0=-1.0)])
    def test_rejects_other(self, kw):
        with pytest.raises(ValueError):
            pd.SolverConfig(**kw)

    def test_echo_keys_match_reference(self):
        from dataclasses import asdict
        assert list(asdict(pd.SolverConfig())) == [
            "tol", "time_limit_s", "restart_mode", "beta", "beta_sufficient", "beta_necessary",
            "beta_artificial", "theta", "eps_zero", "max_iters", "deterministic", "kkt_mode", "kkt_stride",
            "eta0", "omega0"]


class TestScalarRules:
    def test_step_state_relation(self):  # test_pdhg.py:128-132
        step = pd.StepState(eta=0.3, omega=4.0)
        assert step.tau * step.sigma == pytest.approx(step.eta ** 2, rel=1e-15)
        assert step.tau == pytest.approx(0.075)
        assert step.sigma == pytest.approx(1.2)

    def test_primal_weight(self):  # test_pdhg.py:135-144
        assert pd.primal_weight_update(1.0, 4.0, 1.0, theta=0.5) == pytest.approx(2.0, rel=1e-15)
        assert pd.primal_weight_update(1e-12, 4.0, 3.0, eps_zero=1e-10) == 3.0
        assert pd.primal_weight_update(4.0, 1e-12, 3.0, eps_zero=1e-10) == 3.0
        assert pd.primal_weight_update(2.0, 2.0, 1.0, theta=0.5) == pytest.approx(1.0, rel=1e-15)
        with pytest.raises(ValueError):
            pd.primal_weight_update(1.0, 1.0, 0.0)

    def test_should_restart(self):  # test_pdhg.py:166-184
        cfg = pd.SolverConfig()
        assert pd.should_restart(cfg, 0.05, 1.0, 0.01, k=5, total_iterations=1000)
        assert pd.should_restart(cfg, 0.5, 1.0, 0.4, k=5, total_iterations=1000)
        assert not pd.should_restart(cfg, 0.5, 1.0, 0.6, k=5, total_iterations=1000)
        assert pd.should_restart(cfg, 0.95, 1.0, 0.9, k=36, total_iterations=100)
        assert not pd.should_restart(cfg, 0.95, 1.0, 0.9, k=35, total_iterations=100)
        cfg = pd.SolverConfig(restart_mode=pd.FIXED_BETA, beta=0.5)
        assert pd.should_restart(cfg, 0.5, 1.0, 0.0, k=1, total_iterations=2)
        assert not pd.should_restart(cfg, 0.51, 1.0, 0.0, k=1, total_iterations=2)

    def test_eta_rule(self):  # adaptive_stepsize, test_pdhg.py:104-126 with bound 1
        assert eta_from_bound(math.inf, 0.7) == 0.7
        assert eta_from_bound(1.0, 4.0) == pytest.approx(1.0, abs=1e-15)
        assert eta_from_bound(1.0, 0.1) == pytest.approx(0.105)
        assert eta_from_bound(1.0, 0.99) == pytest.approx(1.0)

    def test_default_stepsize(self):  # test_pdhg.py:275-277
        prob = pd.make_problem([[0.0, 1.0], [1.0, 0.0]], [0.5, 0.5], [0.5, 0.5])
        assert pd.default_stepsize(prob) == pytest.approx(0.25)


class TestRecords:
    def test_report_round_trip(self):
        rep = pd.SolveReport(method="pdot", solved=True, wall_time_s=0.0, iterations=3, restarts=1,
                             final_relative_kkt=1e-5, rounded_objective=0.3, duality_gap=1e-7,
                             termination_reason="tolerance", config_echo={"tol": 1e-4},
                             restart_lengths=[2], restart_kkts=[1.0, 0.1])
        assert pd.SolveReport.from_json(rep.to_json()) == rep

    def test_iterate_helpers(self):
        it = pd.Iterate.zeros(2, 3)
        assert it.X.shape == (2, 3) and it.norm() == 0.0
        c = it.copy()
        c.X[0, 0] = 3.0
        assert it.X[0, 0] == 0.0 and c.norm() == 3.0

    def test_problem_container_normalises(self):
        prob = pd.make_problem(np.ones((2, 3)), [1.0, 3.0], [1.0, 1.0, 2.0])
        assert prob.f.tolist() == [0.25, 0.75] and prob.g.sum() == 1.0
        with pytest.raises(pd.InstanceError):
            pd.make_problem(np.ones((2, 2)), [1.0, -1.0], [1.0, 1.0])


class TestShardGeometry:
    """Python mirror (shard.py) == C ABI (pdot_shard_rows) over many shapes; the
    shards tile the rows and align with the 8 reduction groups."""

    def test_python_matches_c(self):
        import ctypes

        from paper_2407_19689_b200 import _lib
        from paper_2407_19689_b200.shard import row_tile, shard_rows
        lib = _lib.load()
        for m, n in [(1024, 1024), (4096, 4096), (16384, 16384), (8192, 32768), (65536, 65536),
                     (2048, 96), (1024, 100000), (3000 * 8 * 16, 700)]:
            tm = row_tile(m, n)
            T = -(-m // tm)
            for R in (1, 2, 4, 8):
                if R > 1 and T % 8:
                    continue
                prev = 0
                for r in range(R):
                    a, b = ctypes.c_int64(), ctypes.c_int64()
                    assert lib.pdot_shard_rows(m, n, R, r, ctypes.byref(a), ctypes.byref(b)) == 0
                    assert (a.value, b.value) == shard_rows(m, n, R, r)
                    assert a.value == prev and (a.value // tm) % (T // 8 if R > 1 else 1) == 0
                    prev = b.value
                assert prev == m

    def test_rejects_bad_shard_counts(self):
        import pytest as _pytest

        from paper_2407_19689_b200.shard import shard_rows
        with _pytest.raises(ValueError):
            shard_rows(1024, 1024, 3, 0)
        with _pytest.raises(ValueError):
            shard_rows(1000, 1000, 2, 0)  # 8 tiles of 128 rows? 1000 rows -> not a multiple of 8 tiles
