"""Multi-process (world size 2 and 4, gloo on CPU) checks of the row-sharded
protocol of SURVEY §8(e) / paper_2407_19689_b200/shard.py:

* every rank derives the same group-aligned row ranges (Python mirror ==
  the C ABI's pdot_shard_rows) and the shards tile the rows exactly;
* the NCCL unique id created by rank 0 through libpdot reaches every rank
  over the torch.distributed group;
* a numpy model of the exchange (each rank sums its own reduction groups in
  tile order, all-gather of the per-group chunks, pairwise combine of the 8
  groups) reproduces the single-process reduction bit for bit - the property
  that makes 1/2/4/8-GPU runs identical.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

TM = 128
GROUPS = 8


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _pair8(g):
    return ((g[0] + g[1]) + (g[2] + g[3])) + ((g[4] + g[5]) + (g[6] + g[7]))


def _group_sum(colpart, g, GS, T):
    acc = np.zeros(colpart.shape[1:])
    for t in range(g * GS, min((g + 1) * GS, T)):
        acc = acc + colpart[t]  # tile order, as group_column_sum in finalize.cu
    return acc


def _single_process_tree(colpart):
    T = colpart.shape[0]
    GS = -(-T // GROUPS)
    groups = [_group_sum(colpart, g, GS, T) for g in range(GROUPS)]
    return _pair8(groups)


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    from paper_2407_19689_b200 import _lib
    from paper_2407_19689_b200.shard import nccl_unique_id, shard_rows

    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    # 1. row ranges
    import ctypes
    lib = _lib.load()
    m_total = 2048
    r0, r1 = ctypes.c_int64(), ctypes.c_int64()
    assert lib.pdot_shard_rows(m_total, 4096, world, rank, ctypes.byref(r0), ctypes.byref(r1)) == 0
    res["rows"] = (r0.value, r1.value)
    res["rows_py"] = shard_rows(m_total, 4096, world, rank)
    # 2. NCCL id broadcast
    res["id"] = nccl_unique_id(None)
    # 3. exchange model: the "global" column partials are seeded identically
    rng = np.random.default_rng(123)
    T, n = m_total // TM, 96
    colpart = rng.standard_normal((T, 4, n)) * np.exp2(rng.integers(-30, 30, (T, 4, n)))
    GS = T // GROUPS
    per = GROUPS // world
    mine = np.stack([_group_sum(colpart, g, GS, T) for g in range(rank * per, (rank + 1) * per)])
    gathered = torch.empty((world * per, 4, n), dtype=torch.float64)
    dist.all_gather_into_tensor(gathered, torch.from_numpy(mine))
    res["combined"] = _pair8([gathered[g].numpy() for g in range(GROUPS)])
    res["single"] = _single_process_tree(colpart)
    dist.barrier()
    dist.destroy_process_group()
    out_q.put((rank, res))


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_protocol_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ranges = [results[r]["rows"] for r in range(world)]
    assert all(results[r]["rows"] == results[r]["rows_py"] for r in range(world))
    assert ranges[0][0] == 0 and ranges[-1][1] == 2048
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
    assert len({results[r]["id"] for r in range(world)}) == 1 and len(results[0]["id"]) == 128
    for r in range(world):
        assert np.array_equal(results[r]["combined"], results[r]["single"])
