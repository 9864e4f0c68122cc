"""``solve``: the restarted-PDHG loop of pdhg.py:254-399 on the device.

The Python side only (1) moves the problem and the start point into HBM,
(2) hands the configuration to ``pdot_solve`` (C ABI), which replays CUDA
graphs of fused passes while the device controller makes every restart /
termination / step-size decision, and (3) turns the device result and the
trace-event ring into the reference's ``(Iterate, SolveReport)``.

With a ``SolveTrace`` that needs iterate snapshots (``restart_points`` are
always recorded by the reference; ``record_inner`` adds every iterate) the
loop advances one pass at a time so the snapshots can be copied out.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import asdict

import numpy as np

from . import _lib
from .config import ADAPTIVE, RELATIVE, SolverConfig, SolveTrace
from .device import DeviceProblem, as_device_problem, detach_handle, get_handle
from .records import Iterate, SolveReport


def config_struct(config: SolverConfig, trace_level: int, poll_passes: int = 0,
                  host_omega: bool = False) -> _lib.Config:
    c = _lib.Config()
    c.tol = config.tol
    c.time_limit_s = config.time_limit_s
    c.beta = config.beta
    c.beta_sufficient = config.beta_sufficient
    c.beta_necessary = config.beta_necessary
    c.beta_artificial = config.beta_artificial
    c.theta = config.theta
    c.eps_zero = config.eps_zero
    c.max_iters = int(config.max_iters)
    c.kkt_stride = int(config.kkt_stride)
    c.adaptive = 1 if config.restart_mode == ADAPTIVE else 0
    c.relative = 1 if config.kkt_mode == RELATIVE else 0
    c.eta0 = -1.0 if config.eta0 is None else float(config.eta0)
    c.omega0 = config.omega0
    c.trace_level = trace_level
    c.poll_passes = poll_passes
    c.host_omega = 1 if host_omega else 0
    return c


def _events(h) -> list:
    out = []
    buf = (_lib.Event * 4096)()
    while True:
        k = h.lib.pdot_get_events(h.ptr, buf, 4096)
        out.extend((buf[i].type, buf[i].ia, buf[i].x, buf[i].y, buf[i].z) for i in range(k))
        if k < 4096:
            return out


class _Prefault:
    """Prepare the host output plan on background threads while the GPU
    iterates.  Default: first-touch fresh pageable pages, so the final
    device->host copy runs at ~19 GB/s instead of ~4 GB/s into untouched
    memory.  PDOT_OUTPUT_PINNED=1 allocates page-locked memory instead (a
    ~49 GB/s DMA), but cudaHostAlloc during the solve stalls the graph
    launches (measured: loop 3.1 s -> 3.8 s at C3), so it is opt-in."""

    def __init__(self, shape, nthreads: int = 16):
        import os
        import threading
        self.shape = shape
        self.arr = None
        self.pinned = os.environ.get("PDOT_OUTPUT_PINNED", "0") == "1"
        if self.pinned:
            self.threads = [threading.Thread(target=self._alloc_pinned, daemon=True)]
        else:
            self.arr = np.empty(shape)
            rows = np.array_split(np.arange(shape[0]), nthreads) if shape[0] else []
            self.threads = [threading.Thread(target=self._touch, args=(r,), daemon=True) for r in rows if len(r)]
        for t in self.threads:
            t.start()

    def _alloc_pinned(self):
        from .device import torch
        self._t = torch.empty(self.shape, dtype=torch.float64, pin_memory=True)
        self.arr = self._t.numpy()

    def _touch(self, r):
        self.arr[r[0]:r[-1] + 1].fill(0.0)

    def result(self):
        for t in self.threads:
            t.join()
        return self.arr


def assemble_report(h, res, config: SolverConfig, trace: SolveTrace | None, round_slot: bool = True):
    """Trace events + device result -> SolveReport (pdhg.py:380-399)."""
    lib = h.lib
    restart_lengths, restart_kkts = [], []
    events = _events(h)
    if trace is not None:
        trace._events = events  # noqa: SLF001 - raw device events (margins for parity reports)
    for typ, ia, x, y, _z in events:
        if typ == _lib.EV_START:
            restart_kkts.append(x)
        elif typ == _lib.EV_RESTART:
            restart_lengths.append(int(ia))
            restart_kkts.append(x)
            if trace is not None:
                trace.restart_kkts.append(x)
                trace.omegas.append(y)
        elif trace is not None and typ == _lib.EV_ACCEPT:
            trace.etas.append(x)
            if ia:
                trace.step_bounds.append(y)
        elif trace is not None and typ == _lib.EV_CAND:
            trace.candidate_kkts.append(x)
    rounded_obj = dual_obj = float("nan")
    if round_slot:
        # rounding + rounded objective on the device (pdhg.py:382-384)
        out = (ctypes.c_double * 3)()
        _lib.check(lib.pdot_round(h.ptr, res.final_slot, None, 0, out))
        rounded_obj, dual_obj = float(out[0]), float(out[1])
    reason = _lib.REASONS.get(res.reason, "unknown")
    report = SolveReport(
        method="pdot",
        solved=reason == "tolerance",
        wall_time_s=0.0 if config.deterministic else float(res.elapsed_s),
        iterations=int(res.iterations),
        restarts=int(res.restarts),
        final_relative_kkt=float(res.final_relative_kkt),
        rounded_objective=rounded_obj,
        duality_gap=abs(rounded_obj - dual_obj),
        termination_reason=reason,
        config_echo=asdict(config),
        restart_lengths=restart_lengths,
        restart_kkts=[float(v) for v in restart_kkts],
    )
    report._passes = int(res.passes)  # noqa: SLF001 - diagnostics for bench/tests
    report._device_s = float(res.device_s)  # noqa: SLF001 - CUDA-event time of the loop
    return report


def solve(prob, config: SolverConfig | None = None, initial: Iterate | None = None,
          trace: SolveTrace | None = None, **kw):
    """Restarted PDHG to the KKT tolerance, iteration or time limit (pdhg.py:254-399);
    see ``_solve`` for the GPU-only keyword options.  The call is one NVTX range
    ("pdot.solve"); libpdot adds ranges for the upload, the loop, rounding and the
    plan copy, so an Nsight timeline shows the phases of every call."""
    from .device import torch
    nvtx = torch.cuda.nvtx if torch is not None else None
    if nvtx is not None:
        nvtx.range_push("pdot.solve")
    try:
        return _solve(prob, config, initial, trace, **kw)
    finally:
        if nvtx is not None:
            nvtx.range_pop()


def _solve(prob, config: SolverConfig | None = None, initial: Iterate | None = None,
           trace: SolveTrace | None = None, *, device: int = 0, return_device: bool = False,
           poll_passes: int = 0, trace_snapshots: bool = True, handle=None, host_omega: bool = False):
    """Run restarted PDHG until the KKT tolerance, iteration or time limit.

    Same contract as the reference ``otsolve.solve`` (pdhg.py:254-265):
    returns the final pre-rounding iterate and a report whose objective and
    duality gap are evaluated on the rounded feasible plan; on a limit the
    best evaluated candidate is returned.  ``prob`` may be a host problem
    (numpy ``C f g``) or a ``DeviceProblem`` already in HBM.  With
    ``return_device=True`` the iterate stays on the device (a ``(slot, handle)``
    pair is returned in place of numpy arrays; see ``solve_device``) and the
    handle is taken out of the shared cache, so no later solve can overwrite
    the returned slot.  ``trace_snapshots=False`` records only the scalar
    trace lists (etas, step bounds, candidate KKTs, omegas, restart KKTs) and
    runs the batched graph loop instead of stepping pass by pass.  ``handle``
    runs the solve on a handle the caller owns (e.g. one returned by an
    earlier ``return_device`` solve) instead of the shared cache.
    ``host_omega=True`` evaluates the primal weight of each adaptive restart on
    the host with libm's exp / log -- the functions the reference's math.exp /
    math.log call (pdhg.py:185) -- instead of CUDA's (which may differ by an
    ulp); the device pauses at each such restart (one round trip).
    GPU-only knobs stay out of SolverConfig so config_echo matches the reference.
    """
    t_start = time.perf_counter()
    phases = {}
    if config is None:
        config = SolverConfig()
    if handle is not None:
        h = handle
    elif isinstance(prob, DeviceProblem):
        h = get_handle(prob.m, prob.n, prob.device)
    else:
        m, n = np.shape(prob.C)
        h = get_handle(m, n, device)
    dp = as_device_problem(prob, device, handle=h)
    if (h.m, h.n, h.device) != (dp.m, dp.n, dp.device):
        raise ValueError("handle shape / device does not match the problem")
    phases["h2d_problem_s"] = time.perf_counter() - t_start
    h.bind(dp)
    if initial is not None:
        h.set_slot(0, initial.X, initial.p, initial.q)
    else:
        h.set_slot(0, None, None, None)
    phases["setup_s"] = time.perf_counter() - t_start - phases["h2d_problem_s"]
    stepwise = trace is not None and (trace_snapshots or trace.record_inner)
    cfg = config_struct(config, trace_level=2 if trace is not None else 0, poll_passes=poll_passes,
                        host_omega=host_omega)
    # dense output plans are pre-faulted during the solve; a screened handle copies
    # only the occupied cells into a zero-filled array (Handle.get_slot)
    out = _Prefault((dp.m, dp.n)) if (not return_device and dp.m * dp.n >= (1 << 22)
                                      and not h.screened()) else None
    res = _lib.Result()
    lib = h.lib
    # wall_time_s counts from the call, as pdhg.py:268 does: the upload and setup
    # above are inside it (elapsed_before), the final KKT and rounding are not
    t_before = time.perf_counter() - t_start
    if not stepwise:
        _lib.check(lib.pdot_solve(h.ptr, ctypes.byref(cfg), t_before, ctypes.byref(res)))
    else:
        _lib.check(lib.pdot_begin(h.ptr, ctypes.byref(cfg), t_before))
        prog = _lib.Progress()
        seen_iter = seen_outer = 0
        avg_duals = []  # dual parts of the averages, known at acceptance (the matrix comes a pass later)
        while True:
            _lib.check(lib.pdot_advance(h.ptr, 1, ctypes.byref(prog)))
            if trace.record_inner and prog.avg_written and avg_duals:
                A, _, _ = h.get_slot(prog.avg_slot)
                pa, qa = avg_duals.pop(0)
                trace.inner_averages.append(Iterate(A, pa, qa))
            if prog.restarts > seen_outer:
                seen_outer = prog.restarts
                X, p, q = h.get_slot(prog.roles[0])
                trace.restart_points.append(Iterate(X, p, q))
            if prog.done:
                break
            if prog.iterations > seen_iter:
                seen_iter = prog.iterations
                if trace.record_inner:
                    X, p, q = h.get_slot(prog.roles[0])
                    trace.inner_iterates.append(Iterate(X, p, q))
                    _, pa, qa = h.get_slot(prog.roles[1], want_X=False)
                    avg_duals.append((pa, qa))
        _lib.check(lib.pdot_finish(h.ptr, ctypes.byref(res)))
    elapsed = time.perf_counter() - t_start
    phases["loop_s"] = float(res.elapsed_s) - t_before

    t1 = time.perf_counter()
    report = assemble_report(h, res, config, trace)
    phases["round_report_s"] = time.perf_counter() - t1
    report._e2e_s = elapsed  # noqa: SLF001
    report._phases = phases  # noqa: SLF001
    if return_device:
        if handle is None:
            detach_handle(h)
        return (int(res.final_slot), h), report
    t2 = time.perf_counter()
    X = None if out is None else out.result()
    phases["prefault_wait_s"] = time.perf_counter() - t2
    X, p, q = h.get_slot(res.final_slot, out=X)
    phases["d2h_plan_s"] = time.perf_counter() - t2 - phases["prefault_wait_s"]
    return Iterate(X, p, q), report


def solve_device(prob: DeviceProblem, config: SolverConfig | None = None, **kw):
    """solve() that leaves the iterate in HBM: returns ((slot, handle), report)."""
    return solve(prob, config, return_device=True, **kw)


def pre_rounding_objective(prob, it: Iterate) -> float:
    """<C, X> of a returned iterate (host helper for reports)."""
    return float(np.vdot(np.asarray(prob.C), it.X))
