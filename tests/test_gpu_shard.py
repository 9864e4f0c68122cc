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


@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_p2p_protocol_concurrent_ranks(nranks):
    """The peer-memory exchange with the ranks genuinely concurrent: R linked
    shard handles' control blocks drive one COOPERATIVE launch, one block per
    rank (co-residency guaranteed; separate launches that spin on each other on
    one GPU are unsafe).  Each rank stores its groups into every rank's buffer,
    releases its flag, acquire-spins on the others' flags, checks all 8 groups
    and consumes the exchange, for 6 rounds (both parities) with rank-staggered
    delays, so the spins really wait."""
    import ctypes

    from paper_2407_19689_b200 import _lib
    from paper_2407_19689_b200.device import Handle
    hs = [Handle(1024, 1024, 0, nranks, r) for r in range(nranks)]
    arr = (ctypes.c_void_p * nranks)(*[h.ptr.value for h in hs])
    _lib.check(hs[0].lib.pdot_p2p_link_local(arr, nranks))
    out = (ctypes.c_ulonglong * (3 * nranks))()
    delay_us = 200.0
    _lib.check(hs[0].lib.pdot_p2p_selftest(arr, nranks, 6, delay_us, out))
    errors = [out[3 * r] for r in range(nranks)]
    waited = [out[3 * r + 1] / 1e3 for r in range(nranks)]
    timeouts = [out[3 * r + 2] for r in range(nranks)]
    print(f"R={nranks}: mismatches {errors}, longest wait per rank (us) {[round(w) for w in waited]}")
    assert errors == [0] * nranks and timeouts == [0] * nranks
    assert max(waited) >= 0.5 * delay_us  # a rank waited for a late peer
    for h in hs:
        h.close()
