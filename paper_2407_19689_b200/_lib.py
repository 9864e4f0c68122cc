"""ctypes binding of libpdot.so (the C ABI declared in include/pdot.h).

The library is built in-tree (``python -m paper_2407_19689_b200.build`` or
``__graft_entry__.build()``) to ``paper_2407_19689_b200/lib/libpdot.so``.
There is deliberately no fallback: if the library or a CUDA device is
missing, every solver entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("PDOT_LIB", Path(__file__).resolve().parent / "lib" / "libpdot.so"))

PDOT_OK = 0
PDOT_EINVAL = -1
PDOT_ECUDA = -2
PDOT_ENONFINITE = -3
PDOT_ELINESEARCH = -4
PDOT_ENCCL = -5
PDOT_ESTATE = -6

REASONS = {1: "tolerance", 2: "iteration_limit", 3: "time_limit"}
EV_START, EV_ACCEPT, EV_CAND, EV_RESTART, EV_REJECT = 1, 2, 3, 4, 5

COST_SQEUCLID_GRID, COST_L1_GRID, COST_L1_RECT = 0, 1, 2

# every symbol include/pdot.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "pdot_last_error", "pdot_version", "pdot_create", "pdot_destroy", "pdot_geometry",
    "pdot_set_problem", "pdot_set_problem_implicit", "pdot_set_slot", "pdot_get_slot", "pdot_slot_ptrs", "pdot_solve",
    "pdot_begin", "pdot_advance", "pdot_finish", "pdot_resume", "pdot_get_events", "pdot_round",
    "pdot_unit_step", "pdot_unit_bound", "pdot_unit_kkt", "pdot_unit_apply_A", "pdot_apply_At",
    "pdot_gen_cost", "pdot_gen_cost_rows", "pdot_fro_norm", "pdot_time_stream_kernel",
    "pdot_kernel_launches", "pdot_time_finalize", "pdot_shard_rows", "pdot_create_shard", "pdot_shard_info",
    "pdot_nccl_unique_id", "pdot_comm_init", "pdot_set_virtual", "pdot_shard_pass", "pdot_exchange_local",
    "pdot_sinkhorn_solve", "pdot_ipc_handle", "pdot_p2p_open", "pdot_p2p_link_local",
    "pdot_set_screening", "pdot_screen_stats", "pdot_get_slot_sparse", "pdot_p2p_selftest",
    "pdot_h2d_matrix", "pdot_shard_pass_ms",
)


class Config(ctypes.Structure):
    _fields_ = [
        ("tol", ctypes.c_double), ("time_limit_s", ctypes.c_double), ("beta", ctypes.c_double),
        ("beta_sufficient", ctypes.c_double), ("beta_necessary", ctypes.c_double),
        ("beta_artificial", ctypes.c_double), ("theta", ctypes.c_double), ("eps_zero", ctypes.c_double),
        ("max_iters", ctypes.c_int64), ("kkt_stride", ctypes.c_int64),
        ("adaptive", ctypes.c_int32), ("relative", ctypes.c_int32),
        ("eta0", ctypes.c_double), ("omega0", ctypes.c_double),
        ("trace_level", ctypes.c_int32), ("poll_passes", ctypes.c_int32),
        ("host_omega", ctypes.c_int32), ("reserved", ctypes.c_int32),
    ]


class Result(ctypes.Structure):
    _fields_ = [
        ("reason", ctypes.c_int32), ("final_slot", ctypes.c_int32),
        ("iterations", ctypes.c_int64), ("restarts", ctypes.c_int64), ("passes", ctypes.c_int64),
        ("rejected", ctypes.c_int64), ("final_relative_kkt", ctypes.c_double), ("eta", ctypes.c_double),
        ("omega", ctypes.c_double), ("scale_R", ctypes.c_double), ("elapsed_s", ctypes.c_double),
        ("device_s", ctypes.c_double),
    ]


class SinkhornCfg(ctypes.Structure):
    _fields_ = [("penalty", ctypes.c_double), ("tol", ctypes.c_double), ("max_iters", ctypes.c_int64),
                ("time_limit_s", ctypes.c_double), ("poll_iters", ctypes.c_int32)]


class Event(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int32), ("ia", ctypes.c_int32), ("x", ctypes.c_double),
                ("y", ctypes.c_double), ("z", ctypes.c_double)]


class Progress(ctypes.Structure):
    _fields_ = [("done", ctypes.c_int32), ("roles", ctypes.c_int32 * 4), ("op", ctypes.c_int32),
                ("iterations", ctypes.c_int64), ("restarts", ctypes.c_int64), ("passes", ctypes.c_int64),
                ("avg_written", ctypes.c_int32), ("avg_slot", ctypes.c_int32)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double
_DP = ctypes.POINTER(ctypes.c_double)

_SIGS = {
    "pdot_last_error": ([], ctypes.c_char_p),
    "pdot_version": ([], ctypes.c_int),
    "pdot_create": ([_I64, _I64, ctypes.c_int, ctypes.POINTER(_P)], ctypes.c_int),
    "pdot_destroy": ([_P], ctypes.c_int),
    "pdot_geometry": ([_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_I64),
                       ctypes.POINTER(_I64)], ctypes.c_int),
    "pdot_set_problem": ([_P, _P, _I64, _P, _P, _D, _D], ctypes.c_int),
    "pdot_set_problem_implicit": ([_P, ctypes.c_int, ctypes.POINTER(_I64), _P, _P, _D, _D], ctypes.c_int),
    "pdot_set_slot": ([_P, ctypes.c_int, _P, _I64, _P, _P], ctypes.c_int),
    "pdot_get_slot": ([_P, ctypes.c_int, _P, _I64, _P, _P], ctypes.c_int),
    "pdot_slot_ptrs": ([_P, ctypes.c_int, ctypes.POINTER(_P), ctypes.POINTER(_P), ctypes.POINTER(_P)],
                       ctypes.c_int),
    "pdot_solve": ([_P, ctypes.POINTER(Config), _D, ctypes.POINTER(Result)], ctypes.c_int),
    "pdot_begin": ([_P, ctypes.POINTER(Config), _D], ctypes.c_int),
    "pdot_advance": ([_P, _I64, ctypes.POINTER(Progress)], ctypes.c_int),
    "pdot_finish": ([_P, ctypes.POINTER(Result)], ctypes.c_int),
    "pdot_resume": ([_P, _I64, ctypes.POINTER(Result)], ctypes.c_int),
    "pdot_get_events": ([_P, ctypes.POINTER(Event), _I64], _I64),
    "pdot_round": ([_P, ctypes.c_int, _P, _I64, _DP], ctypes.c_int),
    "pdot_unit_step": ([_P, _D, _D, _D], ctypes.c_int),
    "pdot_unit_bound": ([_P, _D, _D, _DP], ctypes.c_int),
    "pdot_unit_kkt": ([_P, _D, _P, _I64, _P, _P, _DP], ctypes.c_int),
    "pdot_unit_apply_A": ([_P, _P, _P], ctypes.c_int),
    "pdot_apply_At": ([_P, _P, _I64, _I64, _P, _I64], ctypes.c_int),
    "pdot_gen_cost": ([_P, _I64, _I64, _I64, ctypes.c_int, ctypes.POINTER(_I64)], ctypes.c_int),
    "pdot_fro_norm": ([_P, _I64, _I64, _I64, _DP], ctypes.c_int),
    "pdot_shard_pass_ms": ([_P, _DP], ctypes.c_int),
    "pdot_h2d_matrix": ([_P, _I64, _P, _I64, _I64, _I64, ctypes.c_int], ctypes.c_int),
    "pdot_time_stream_kernel": ([_P, ctypes.c_int, _DP], ctypes.c_int),
    "pdot_kernel_launches": ([_P], _I64),
    "pdot_time_finalize": ([_P, ctypes.c_int, _DP], ctypes.c_int),
    "pdot_gen_cost_rows": ([_P, _I64, _I64, _I64, _I64, ctypes.c_int, ctypes.POINTER(_I64)], ctypes.c_int),
    "pdot_shard_rows": ([_I64, _I64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_I64), ctypes.POINTER(_I64)],
                        ctypes.c_int),
    "pdot_create_shard": ([_I64, _I64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)],
                          ctypes.c_int),
    "pdot_shard_info": ([_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(ctypes.c_int32),
                         ctypes.POINTER(ctypes.c_int32)], ctypes.c_int),
    "pdot_nccl_unique_id": ([_P], ctypes.c_int),
    "pdot_comm_init": ([_P, _P], ctypes.c_int),
    "pdot_set_virtual": ([_P, ctypes.c_int], ctypes.c_int),
    "pdot_shard_pass": ([_P, ctypes.c_int, ctypes.POINTER(Progress)], ctypes.c_int),
    "pdot_exchange_local": ([ctypes.POINTER(_P), ctypes.c_int], ctypes.c_int),
    "pdot_sinkhorn_solve": ([_P, ctypes.POINTER(SinkhornCfg), _D, ctypes.POINTER(Result)], ctypes.c_int),
    "pdot_ipc_handle": ([_P, _P], ctypes.c_int),
    "pdot_p2p_open": ([_P, _P, ctypes.c_int], ctypes.c_int),
    "pdot_p2p_link_local": ([ctypes.POINTER(_P), ctypes.c_int], ctypes.c_int),
    "pdot_p2p_selftest": ([ctypes.POINTER(_P), ctypes.c_int, ctypes.c_int, _D, ctypes.POINTER(ctypes.c_ulonglong)],
                          ctypes.c_int),
    "pdot_set_screening": ([_P, ctypes.c_int], ctypes.c_int),
    "pdot_get_slot_sparse": ([_P, ctypes.c_int, _P, _I64, _P, _P, ctypes.POINTER(_I64)], ctypes.c_int),
    "pdot_screen_stats": ([_P, ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong)], ctypes.c_int),
}

_lib = None


def load(path: Path | None = None):
    """Load libpdot.so once; raise loudly when it is missing (no fallback)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else Path(os.environ.get("PDOT_LIB_PATH") or LIB_PATH)
    if not p.exists():
        raise RuntimeError(
            f"libpdot.so not found at {p}: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the PDOT solver has no CPU fallback)")
    lib = ctypes.CDLL(str(p))
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if path is None:
        _lib = lib
    return lib


def last_error() -> str:
    return load().pdot_last_error().decode(errors="replace")


def check(rc: int) -> None:
    """Map a PDOT status to the reference's exception types (include/pdot.h)."""
    if rc == PDOT_OK:
        return
    msg = last_error()
    if rc == PDOT_EINVAL:
        raise ValueError(msg)
    if rc == PDOT_ENONFINITE:
        raise RuntimeError(msg if "potential" in msg else "numerical failure: non-finite iterate")
    if rc == PDOT_ELINESEARCH:
        raise RuntimeError("step-size line search failed to find an admissible eta")
    raise RuntimeError(f"libpdot error {rc}: {msg}")
