"""Device residency: problems on the GPU and cached solver handles.

PyTorch is used only as the device allocator and for host<->device copies;
all arithmetic on the path runs in libpdot.so's kernels.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None


def require_cuda(device: int = 0) -> None:
    if torch is None or not torch.cuda.is_available():
        raise RuntimeError("PDOT needs a CUDA device: there is no CPU fallback")
    if device >= torch.cuda.device_count():
        raise RuntimeError(f"CUDA device {device} not present")


def even(n: int) -> int:
    return n + (n & 1)


def _h2d_matrix(A: np.ndarray, device: int, out=None):
    """Host -> HBM copy of the cost matrix through ``pdot_h2d_matrix``: one
    direct DMA from page-locked memory, or, from pageable memory (a plain numpy
    array), a pinned double buffer filled by host threads while the other half
    is DMA'd (csrc/solver.cu).  Odd n gets a zero pad column (even ldc)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    m, n = A.shape
    if out is not None and tuple(out.shape) == (m, even(n)):
        t = out  # a buffer the caller owns (the handle's cost buffer): no 2 GB allocation per call
    else:
        t = (torch.empty((m, n), dtype=torch.float64, device=f"cuda:{device}") if n % 2 == 0
             else torch.zeros((m, n + 1), dtype=torch.float64, device=f"cuda:{device}"))
    torch.cuda.synchronize(device)
    _lib.check(_lib.load().pdot_h2d_matrix(t.data_ptr(), t.stride(0), A.ctypes.data, n, m, n, device))
    return t


def _h2d_vector(v: np.ndarray, device: int):
    return torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(f"cuda:{device}")


class DeviceProblem:
    """An OT problem resident in HBM: C (m x ldc, ldc even), f (m), g (n).

    Exposes the OTProblem accessors the solver needs (m, n, cost_fro_norm,
    marginal_norm; instance.py:122-150).  ``host`` keeps the originating host
    problem when there is one.
    """

    def __init__(self, C_t, f_t, g_t, m, n, cost_fro_norm, marginal_norm, device=0, host=None):
        self.C_t, self.f_t, self.g_t = C_t, f_t, g_t
        self.m, self.n = int(m), int(n)
        self.cost_fro_norm = float(cost_fro_norm)
        self.marginal_norm = float(marginal_norm)
        self.device = device
        self.host = host
        self.m_total, self.row0 = self.m, 0
        self.cost_kind, self.cost_args = None, None

    @property
    def ldc(self) -> int:
        return int(self.C_t.stride(0)) if self.C_t is not None else even(self.n)

    @property
    def implicit(self) -> bool:
        """True when C is generated in-kernel from grid coordinates (no cost buffer)."""
        return self.C_t is None

    @classmethod
    def from_host(cls, prob, device: int = 0, out=None) -> "DeviceProblem":
        """Upload a host problem; ``out`` (an (m, even n) float64 CUDA tensor) receives C
        instead of a fresh allocation."""
        require_cuda(device)
        C = np.asarray(prob.C, dtype=np.float64)
        return cls(_h2d_matrix(C, device, out), _h2d_vector(prob.f, device), _h2d_vector(prob.g, device),
                   C.shape[0], C.shape[1], prob.cost_fro_norm, prob.marginal_norm, device, host=prob)

    @classmethod
    def generated(cls, kind: int, m: int, n: int, shape_args, f: np.ndarray, g: np.ndarray,
                  device: int = 0, fro: float | None = None, rows=None, implicit: bool = False) -> "DeviceProblem":
        """Cost built on the device (pdot_gen_cost_rows), marginals from the host.

        ``rows = (row0, row1)`` builds only that row shard (C rows and f entries);
        ``fro`` is the exact ||C||_F of the FULL matrix (instances.*_fro_norm),
        so every shard and GPU count sees the same KKT normaliser.  With
        ``implicit=True`` no cost buffer is allocated: the kernels generate C_ij
        from grid coordinates (matrix-free variant)."""
        require_cuda(device)
        lib = _lib.load()
        row0, row1 = (0, m) if rows is None else rows
        C_t = None
        if not implicit:
            C_t = torch.empty((row1 - row0, even(n)), dtype=torch.float64, device=f"cuda:{device}")
            args = (ctypes.c_int64 * 4)(*shape_args)
            torch.cuda.synchronize(device)
            _lib.check(lib.pdot_gen_cost_rows(C_t.data_ptr(), row0, row1 - row0, n, C_t.stride(0), kind, args))
        if fro is None:
            if rows is not None or implicit:
                raise ValueError("a row shard / implicit cost needs the exact full-matrix Frobenius norm")
            out = ctypes.c_double()
            _lib.check(lib.pdot_fro_norm(C_t.data_ptr(), m, n, C_t.stride(0), ctypes.byref(out)))
            fro = out.value
        marg = float(np.linalg.norm(f) + np.linalg.norm(g))
        dp = cls(C_t, _h2d_vector(f[row0:row1], device), _h2d_vector(g, device), row1 - row0, n, fro, marg,
                 device)
        dp.m_total, dp.row0 = m, row0
        dp.cost_kind, dp.cost_args = kind, tuple(shape_args)
        return dp

    @classmethod
    def sqeuclid_grid(cls, r: int, seed: int, device: int = 0, rows=None, implicit: bool = False) -> "DeviceProblem":
        """Configs C1/C2/C3/C5: whitenoise marginals, exact squared-Euclidean grid cost."""
        from .instances import sqeuclid_fro_norm, whitenoise_marginals
        f, g = whitenoise_marginals(r, seed)
        return cls.generated(_lib.COST_SQEUCLID_GRID, r * r, r * r, (r, r, 0, 0), f, g, device,
                             fro=sqeuclid_fro_norm(r), rows=rows, implicit=implicit)

    @classmethod
    def rect_l1(cls, seed: int, src=(64, 128), dst=(128, 256), device: int = 0, rows=None,
                implicit: bool = False) -> "DeviceProblem":
        """Config C4: rectangular L1 cost with sparse-support marginals."""
        from .instances import rect_l1_fro_norm, sparse_marginals
        m, n = src[0] * src[1], dst[0] * dst[1]
        f = sparse_marginals(m, 2 * seed)
        g = sparse_marginals(n, 2 * seed + 1)
        return cls.generated(_lib.COST_L1_RECT, m, n, (src[0], src[1], dst[0], dst[1]), f, g, device,
                             fro=rect_l1_fro_norm(src, dst), rows=rows, implicit=implicit)

    def row_shard(self, row0: int, row1: int) -> "DeviceProblem":
        """View of rows [row0, row1) of this (full) problem: C rows and f entries."""
        C = None if self.C_t is None else self.C_t[row0:row1]
        dp = DeviceProblem(C, self.f_t[row0:row1], self.g_t, row1 - row0, self.n,
                           self.cost_fro_norm, self.marginal_norm, self.device)
        dp.m_total, dp.row0 = self.m, row0
        dp.cost_kind, dp.cost_args = self.cost_kind, self.cost_args
        return dp


def as_device_problem(prob, device: int = 0, handle=None) -> DeviceProblem:
    """A host problem goes to HBM; with a handle, into that handle's reusable cost
    buffer (repeated solve() calls of one shape then allocate nothing)."""
    if isinstance(prob, DeviceProblem):
        return prob
    out = handle.cost_buffer() if handle is not None else None
    return DeviceProblem.from_host(prob, device, out=out)


def zeros_plan(shape):
    """A zero-filled float64 array whose untouched pages stay the shared zero
    page: anonymous memory with 4 KB pages (numpy's own large allocations ask
    for 2 MB pages, and every first touch of one zeroes 2 MB -- scattering a
    sparse plan into np.zeros of a 16384^2 plan costs ~35 ms, into this ~5 ms)."""
    import mmap
    nbytes = int(np.prod(shape)) * 8
    if nbytes < (1 << 22):
        return np.zeros(shape)
    mm = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    if hasattr(mmap, "MADV_NOHUGEPAGE"):
        mm.madvise(mmap.MADV_NOHUGEPAGE)
    return np.frombuffer(mm, dtype=np.float64).reshape(shape)


class Handle:
    """Owns one pdot_solver* (one problem shape, or one row shard, on one GPU)."""

    def __init__(self, m: int, n: int, device: int = 0, nranks: int = 1, rank: int = 0):
        require_cuda(device)
        torch.cuda.init()
        self.lib = _lib.load()
        ptr = ctypes.c_void_p()
        _lib.check(self.lib.pdot_create_shard(m, n, nranks, rank, device, ctypes.byref(ptr)))
        self.ptr = ptr
        self.nranks, self.rank, self.m_total = nranks, rank, m
        if nranks > 1:
            r0, r1 = ctypes.c_int64(), ctypes.c_int64()
            _lib.check(self.lib.pdot_shard_rows(m, n, nranks, rank, ctypes.byref(r0), ctypes.byref(r1)))
            self.row0, m = r0.value, r1.value - r0.value
        else:
            self.row0 = 0
        self.m, self.n, self.device = m, n, device
        ldx = ctypes.c_int64()
        _lib.check(self.lib.pdot_geometry(ptr, ctypes.byref(ldx), None, None, None))
        self.ldx = ldx.value
        self.bytes = 6 * 8 * m * self.ldx
        self.bound_problem = None
        self.screen = None  # None: the library default (PDOT_SCREEN, on unless set to 0)

    def close(self):
        if self.ptr:
            self.lib.pdot_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def bind(self, dp: DeviceProblem) -> None:
        torch.cuda.synchronize(dp.device)
        if dp.implicit:
            args = (ctypes.c_int64 * 4)(*dp.cost_args)
            _lib.check(self.lib.pdot_set_problem_implicit(self.ptr, dp.cost_kind, args, dp.f_t.data_ptr(),
                                                          dp.g_t.data_ptr(), dp.cost_fro_norm, dp.marginal_norm))
        else:
            _lib.check(self.lib.pdot_set_problem(self.ptr, dp.C_t.data_ptr(), dp.ldc, dp.f_t.data_ptr(),
                                                 dp.g_t.data_ptr(), dp.cost_fro_norm, dp.marginal_norm))
        self.bound_problem = dp  # keep the borrowed buffers alive
        if _SCREEN is not None and _SCREEN != self.screen:
            self.set_screening(_SCREEN)

    def set_screening(self, on: bool) -> None:
        """Block screening of the STEP pass (bit-identical results)."""
        _lib.check(self.lib.pdot_set_screening(self.ptr, 1 if on else 0))
        self.screen = bool(on)

    def screen_stats(self, reset: bool = False) -> dict:
        out = (ctypes.c_ulonglong * 20)()
        _lib.check(self.lib.pdot_screen_stats(self.ptr, 1 if reset else 0, out))
        keys = ("passes", "active_cells", "cells_visited", "k1_bytes", "k0_bytes", "k1_ns", "screen_on",
                "cells_per_plan", "k2_main_ns", "k2_ctl_ns", "ctl_reduce_ns", "ctl_logic_ns", "ctl_publish_ns",
                "gap_k2_k0_ns", "k0_to_k1_ns", "k1_to_k2_ns", "gap_k2_k0_entry_ns")
        return dict(zip(keys, (int(v) for v in out)))

    def set_slot(self, slot: int, X=None, p=None, q=None) -> None:
        keep = []

        def ptr(a, shape):
            if a is None:
                return None, 0
            if torch is not None and isinstance(a, torch.Tensor):
                if tuple(a.shape) != shape:
                    raise ValueError("shape mismatch")
                t = a.to(dtype=torch.float64)
                if t.dim() == 2 and t.stride(1) != 1:
                    t = t.contiguous()
                keep.append(t)
                return t.data_ptr(), (t.stride(0) if t.dim() == 2 else 0)
            arr = np.ascontiguousarray(a, dtype=np.float64)
            if arr.shape != shape:
                raise ValueError(f"shape mismatch: expected {shape}, got {arr.shape}")
            keep.append(arr)
            return arr.ctypes.data, (arr.shape[1] if arr.ndim == 2 else 0)

        Xp, ld = ptr(X, (self.m, self.n))
        pp, _ = ptr(p, (self.m,))
        qp, _ = ptr(q, (self.n,))
        if keep and torch is not None:
            torch.cuda.synchronize(self.device)
        _lib.check(self.lib.pdot_set_slot(self.ptr, slot, Xp, ld if Xp else self.n, pp, qp))

    def cost_buffer(self):
        """The handle's own (m, even n) device buffer for uploaded cost matrices."""
        if getattr(self, "_cbuf", None) is None:
            z = torch.empty if self.n % 2 == 0 else torch.zeros
            self._cbuf = z((self.m, even(self.n)), dtype=torch.float64, device=f"cuda:{self.device}")
        return self._cbuf

    def screened(self) -> bool:
        return self.screen_stats()["screen_on"] == 1

    def get_slot(self, slot: int, want_X=True, out=None):
        """Copy a slot to the host.  On a screened handle only the occupied 8x16
        cells travel (every other cell is exactly +0.0 on the device) into a
        zero-filled array; otherwise the dense plan is copied."""
        p = np.empty(self.m)
        q = np.empty(self.n)
        if want_X and out is None and self.screened():
            X = zeros_plan((self.m, self.n))
            cells = ctypes.c_int64()
            _lib.check(self.lib.pdot_get_slot_sparse(self.ptr, slot, X.ctypes.data, self.n, p.ctypes.data,
                                                     q.ctypes.data, ctypes.byref(cells)))
            return X, p, q
        X = (out if out is not None else np.empty((self.m, self.n))) if want_X else None
        _lib.check(self.lib.pdot_get_slot(self.ptr, slot, X.ctypes.data if want_X else None, self.n,
                                          p.ctypes.data, q.ctypes.data))
        return X, p, q

    def launches(self) -> int:
        return int(self.lib.pdot_kernel_launches(self.ptr))


_HANDLES: dict = {}
_BIG = 1 << 30
_SCREEN = None


def set_screening(on) -> None:
    """Process-wide override of block screening for handles bound from now on:
    True / False, or None for the library default (on; PDOT_SCREEN=0 turns it
    off).  Results are bit-identical either way; tests flip it to prove that."""
    global _SCREEN
    _SCREEN = None if on is None else bool(on)


def get_handle(m: int, n: int, device: int = 0) -> Handle:
    key = (m, n, device)
    h = _HANDLES.get(key)
    if h is not None:
        return h
    need = 6 * 8 * m * even(n)
    if need > _BIG or sum(x.bytes for x in _HANDLES.values()) > 4 * _BIG or len(_HANDLES) > 32:
        release_handles()
    h = Handle(m, n, device)
    _HANDLES[key] = h
    return h


def detach_handle(h: Handle) -> None:
    """Take ``h`` out of the shared cache: its caller now owns it exclusively
    (a device-resident result in one of its slots cannot be overwritten by a
    later solve of the same shape, which gets a fresh handle)."""
    for k, v in list(_HANDLES.items()):
        if v is h:
            del _HANDLES[k]


def release_handles() -> None:
    """Drop the cache's references; a handle is destroyed once no caller holds
    it (a solve_device result keeps its handle alive)."""
    import gc
    _HANDLES.clear()
    gc.collect()
    if torch is not None and torch.cuda.is_available():
        torch.cuda.empty_cache()
