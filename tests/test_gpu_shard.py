"""Row sharding on one GPU: R shard handles stepped together
with device-copy exchanges must reproduce the single-GPU solve BIT FOR BIT
(same reduction tree), for R = 2, 4, 8."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("transport", ["copy", "p2p"])
@pytest.mark.parametrize("nshards", [2, 4, 8])
def test_virtual_shards_bit_identical(nshards, transport):
    import paper_2407_19689_b200 as pd
    from paper_2407_19689_b200.shard import solve_virtual
    dp = pd.DeviceProblem.sqeuclid_grid(32, 1)  # C1 family, m = n = 1024 (8 row tiles)
    cfg = pd.SolverConfig(tol=1e-4, deterministic=True)
    it1, rep1 = pd.solve(dp, cfg)
    itv, repv = solve_virtual(dp, cfg, nshards, transport=transport)
    assert repv.iterations == rep1.iterations and repv.restarts == rep1.restarts
    assert repv.restart_lengths == rep1.restart_lengths
    assert repv.restart_kkts == rep1.restart_kkts
    assert repv.final_relative_kkt == rep1.final_relative_kkt
    assert np.array_equal(itv.X, it1.X)
    assert np.array_equal(itv.p, it1.p) and np.array_equal(itv.q, it1.q)


def test_virtual_shards_rectangular_limit():
    import paper_2407_19689_b200 as pd
    from paper_2407_19689_b200.shard import solve_virtual
    dp = pd.DeviceProblem.rect_l1(0, src=(32, 64), dst=(64, 128))  # m = 2048 (16 tiles), n = 8192
    cfg = pd.SolverConfig(tol=1e-9, max_iters=60, deterministic=True)
    it1, rep1 = pd.solve(dp, cfg)
    itv, repv = solve_virtual(dp, cfg, 4, transport="p2p")
    assert rep1.termination_reason == repv.termination_reason == "iteration_limit"
    assert repv.iterations == rep1.iterations == 60
    assert np.array_equal(itv.X, it1.X)
    assert np.array_equal(itv.p, it1.p) and np.array_equal(itv.q, it1.q)
