"""The multi-GPU pass sequence (stream -> group partials -> ncclAllGather ->
combine + controller), replayed from captured CUDA graphs exactly as a
row-sharded run does, on ONE GPU through a 1-rank NCCL communicator
(PDOT_FORCE_SPLIT=1).  Must be bit-identical to the fused single-GPU path."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_split_sequence_with_nccl_matches_fused():
    import paper_2407_19689_b200 as pd
    from paper_2407_19689_b200.shard import ShardedSolver
    dp = pd.DeviceProblem.sqeuclid_grid(32, 2)
    cfg = pd.SolverConfig(tol=1e-5, deterministic=True)
    it1, rep1 = pd.solve(dp, cfg)
    os.environ["PDOT_FORCE_SPLIT"] = "1"
    try:
        solver = ShardedSolver(dp.row_shard(0, dp.m), 1, 0)
        res, rep2 = solver.solve(cfg)
        it2 = solver.local_iterate()
        solver.close()
    finally:
        del os.environ["PDOT_FORCE_SPLIT"]
    assert rep2.iterations == rep1.iterations and rep2.restarts == rep1.restarts
    assert rep2.restart_kkts == rep1.restart_kkts
    assert rep2.final_relative_kkt == rep1.final_relative_kkt
    assert rep2.rounded_objective == rep1.rounded_objective
    assert np.array_equal(it2.X, it1.X) and np.array_equal(it2.p, it1.p) and np.array_equal(it2.q, it1.q)


def test_split_sequence_screened_c2():
    """The same at C2 (4096^2 = 2^24 entries, screened passes by default): K0 /
    K1 / K1b, then FIN_A group partials -> ncclAllGather (1-rank communicator)
    -> FIN_B combine + controller, from captured graphs; bit-identical to the
    fused screened pass over 300 iterations."""
    import paper_2407_19689_b200 as pd
    from paper_2407_19689_b200.device import get_handle
    from paper_2407_19689_b200.shard import ShardedSolver
    dp = pd.DeviceProblem.sqeuclid_grid(64, 0)
    cfg = pd.SolverConfig(tol=1e-9, deterministic=True, max_iters=300)
    it1, rep1 = pd.solve(dp, cfg)
    assert get_handle(dp.m, dp.n).screened()
    os.environ["PDOT_FORCE_SPLIT"] = "1"
    try:
        solver = ShardedSolver(dp.row_shard(0, dp.m), 1, 0)
        assert solver.h.screened()
        res, rep2 = solver.solve(cfg)
        it2 = solver.local_iterate()
        solver.close()
    finally:
        del os.environ["PDOT_FORCE_SPLIT"]
    assert (rep2.iterations, rep2.restarts, rep2.restart_lengths) == (rep1.iterations, rep1.restarts,
                                                                       rep1.restart_lengths)
    assert rep2.restart_kkts == rep1.restart_kkts
    assert rep2.final_relative_kkt == rep1.final_relative_kkt
    assert np.array_equal(it2.X, it1.X) and np.array_equal(it2.p, it1.p) and np.array_equal(it2.q, it1.q)
