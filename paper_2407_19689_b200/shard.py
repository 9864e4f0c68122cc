"""Row-sharded solve over several GPUs.

Shard r of R owns rows [row0, row1) of C, X, the running average, the anchor
and the best point, and the matching entries of f and p; q and g are
replicated.  Row boundaries follow the 8-group reduction tree of the
finalize kernel (``pdot_shard_rows``), so each shard computes whole groups of
every reduction and one all-gather per pass hands every shard all 8 groups:
the combine, the q-update and the controller then run identically on every
GPU, and the iterates are bit-identical to the single-GPU solve (checked by
``tests/test_gpu_shard.py`` with the single-GPU emulation below).

Transports:
* ``nccl`` (default): ``ncclAllGather`` (torch's libnccl, over NVLink/NVSwitch)
  issued by libpdot on its own stream inside the captured CUDA graph; the
  unique id travels over the caller's ``torch.distributed`` group.
* ``p2p``: the finalize kernel itself stores its group partials into every
  rank's exchange buffer (CUDA IPC-mapped peer memory) and publishes a
  sequence flag with release semantics; the combine kernel acquires all flags.
  The collective is fused into the compute kernel; no NCCL call per pass.
For tests on one GPU, ``solve_virtual`` steps R shard handles on the same
device: ``copy`` moves the exchange buffers with device copies, ``p2p`` runs
the peer-store path with the handles linked to each other (every writer
completes before any reader starts, so no kernel ever waits on another).
"""

from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _lib
from .config import SolverConfig
from .device import DeviceProblem, Handle
from .engine import assemble_report, config_struct
from .records import Iterate

GROUPS = 8


def row_tile(m_total: int, n: int) -> int:
    """Rows per streaming tile (mirror of row_tile() in csrc/solver.cu)."""
    import os
    tm = 128
    u = -(-n // 512)
    while tm > 16 and -(-m_total // tm) * u < 148:
        tm //= 2
    env = os.environ.get("PDOT_TM")
    if env is not None:
        tm = int(env) if int(env) in (8, 16, 32, 64, 128, 256) else 128
    return tm


def shard_rows(m_total: int, n: int, nranks: int, rank: int):
    """Group-aligned row range of a shard (pure-Python mirror of pdot_shard_rows)."""
    row_tile_ = row_tile(m_total, n)
    T = -(-m_total // row_tile_)
    if nranks not in (1, 2, 4, 8):
        raise ValueError("row sharding supports 1, 2, 4 or 8 shards")
    if not 0 <= rank < nranks:
        raise ValueError("rank out of range")
    if nranks > 1 and T % GROUPS:
        raise ValueError("row sharding needs the number of row tiles to be a multiple of 8")
    gs = -(-T // GROUPS)
    per = GROUPS // nranks
    t0, t1 = min(rank * per * gs, T), min((rank + 1) * per * gs, T)
    return min(t0 * row_tile_, m_total), min(t1 * row_tile_, m_total)


def _bind_shard(h: Handle, dp: DeviceProblem) -> None:
    if dp.m != h.m or dp.row0 != h.row0:
        raise ValueError("problem shard does not match the handle's row range")
    h.bind(dp)


def solve_virtual(dp: DeviceProblem, config: SolverConfig | None = None, nshards: int = 2,
                  initial: Iterate | None = None, transport: str = "copy"):
    """Single-GPU emulation of an R-shard solve (test path).

    Returns the gathered full iterate and the report of shard 0.  Every shard
    must reach identical decisions; this is asserted pass by pass.
    """
    if config is None:
        config = SolverConfig()
    m, n = dp.m, dp.n
    hs = [Handle(m, n, dp.device, nshards, r) for r in range(nshards)]
    for h in hs:
        _bind_shard(h, dp.row_shard(h.row0, h.row0 + h.m))
        _lib.check(h.lib.pdot_set_virtual(h.ptr, 1))
        if initial is None:
            h.set_slot(0, None, None, None)
        else:
            sl = slice(h.row0, h.row0 + h.m)
            h.set_slot(0, initial.X[sl], initial.p[sl], initial.q)
    arr = (ctypes.c_void_p * nshards)(*[h.ptr.value for h in hs])
    if transport == "p2p":
        _lib.check(hs[0].lib.pdot_p2p_link_local(arr, nshards))
    elif transport != "copy":
        raise ValueError(f"unknown transport {transport!r}")
    cfg = config_struct(config, trace_level=0)
    for h in hs:
        _lib.check(h.lib.pdot_begin(h.ptr, ctypes.byref(cfg), 0.0))
    progs = [_lib.Progress() for _ in hs]
    lib = hs[0].lib
    while True:
        for h in hs:
            _lib.check(lib.pdot_shard_pass(h.ptr, 0, None))
        if transport == "copy":
            _lib.check(lib.pdot_exchange_local(arr, nshards))
        for h, pr in zip(hs, progs):
            _lib.check(lib.pdot_shard_pass(h.ptr, 1, ctypes.byref(pr)))
        state = {(p.done, p.iterations, p.restarts, p.passes, tuple(p.roles)) for p in progs}
        if len(state) != 1:
            raise RuntimeError(f"shards diverged: {state}")
        if progs[0].done:
            break
    results = []
    for h in hs:
        res = _lib.Result()
        _lib.check(lib.pdot_finish(h.ptr, ctypes.byref(res)))
        results.append(res)
    X = np.empty((m, n))
    p = np.empty(m)
    q = None
    for h, res in zip(hs, results):
        Xs, ps, qs = h.get_slot(res.final_slot)
        X[h.row0:h.row0 + h.m] = Xs
        p[h.row0:h.row0 + h.m] = ps
        if q is None:
            q = qs
    report = assemble_report(hs[0], results[0], config, None, round_slot=False)
    for h in hs:
        h.close()
    return Iterate(X, p, q), report


def nccl_unique_id(group=None) -> bytes:
    """Rank 0 creates the NCCL id; every rank of `group` receives it."""
    import torch.distributed as dist

    lib = _lib.load()
    buf = (ctypes.c_char * 128)()
    obj = [None]
    if dist.get_rank(group) == 0:
        _lib.check(lib.pdot_nccl_unique_id(buf))
        obj = [bytes(buf.raw)]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                               group=group)
    return obj[0]


class ShardedSolver:
    """One rank of a row-sharded solve (one process per GPU).

    ``dp`` is this rank's row shard (``DeviceProblem.sqeuclid_grid(...,
    rows=shard_rows(...))`` or ``full.row_shard(...)``).
    """

    def __init__(self, dp: DeviceProblem, nranks: int, rank: int, group=None, transport: str | None = None):
        import os
        self.h = Handle(dp.m_total, dp.n, dp.device, nranks, rank)
        _bind_shard(self.h, dp)
        self.transport = transport or os.environ.get("PDOT_EXCHANGE", "nccl")
        if self.transport == "p2p" and nranks > 1:
            self._open_p2p(group)
            self.dp = dp
            return
        if nranks == 1:  # a 1-rank communicator (PDOT_FORCE_SPLIT tests the split pass sequence)
            buf = (ctypes.c_char * 128)()
            _lib.check(self.h.lib.pdot_nccl_unique_id(buf))
            ident = bytes(buf.raw)
        else:
            ident = nccl_unique_id(group)
        idbuf = ctypes.create_string_buffer(ident, 128)
        _lib.check(self.h.lib.pdot_comm_init(self.h.ptr, idbuf))
        self.dp = dp

    def _open_p2p(self, group):
        """Share every rank's exchange buffer through CUDA IPC handles."""
        import torch.distributed as dist
        buf = (ctypes.c_char * 64)()
        _lib.check(self.h.lib.pdot_ipc_handle(self.h.ptr, buf))
        handles = [None] * self.h.nranks
        dist.all_gather_object(handles, bytes(buf.raw), group=group)
        joined = ctypes.create_string_buffer(b"".join(handles), 64 * self.h.nranks)
        _lib.check(self.h.lib.pdot_p2p_open(self.h.ptr, joined, self.h.nranks))

    def solve(self, config: SolverConfig | None = None, initial: Iterate | None = None):
        """Local rows of the final iterate (+ replicated q) and the report."""
        t0 = time.perf_counter()
        if config is None:
            config = SolverConfig()
        h = self.h
        if initial is None:
            h.set_slot(0, None, None, None)
        else:
            h.set_slot(0, initial.X, initial.p, initial.q)
        cfg = config_struct(config, trace_level=0)
        res = _lib.Result()
        _lib.check(h.lib.pdot_solve(h.ptr, ctypes.byref(cfg), time.perf_counter() - t0, ctypes.byref(res)))
        report = assemble_report(h, res, config, None, round_slot=True)
        self.result = res
        return res, report

    def local_iterate(self):
        X, p, q = self.h.get_slot(self.result.final_slot)
        return Iterate(X, p, q)

    def close(self):
        self.h.close()
