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
