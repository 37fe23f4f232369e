"""B200-native SymmSpMV (arXiv 1907.06487, RACE) — thin Python binding.

Argument marshalling only: every step of the hot path runs inside
``libsymmspmv.so`` (include/symmspmv.h): the RACE schedule builder (C++) and
the sm_100a kernels.  There is no CPU fallback; importing this package fails
loudly when the native library is missing.  PyTorch is used only for device
memory, streams and ``torch.distributed``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from ._lib import (SYMM_ORDER_ORIGINAL, SYMM_ORDER_PERMUTED, VARIANTS, SymmError, check, lib)

__all__ = ["build_schedule", "Schedule", "Plan", "Sweep", "bw_probe", "VARIANTS", "SymmError", "min_bytes", "flops",
           "SYMM_ORDER_PERMUTED", "SYMM_ORDER_ORIGINAL", "library_path"]

library_path = _lib.LIB_PATH


def _csr_struct(U):
    rp = np.ascontiguousarray(U.row_ptr, dtype=np.int32)
    col = np.ascontiguousarray(U.col, dtype=np.int32)
    val = np.ascontiguousarray(U.val, dtype=np.float64)
    s = _lib.SymmCsrUpper(int(U.n), int(rp[-1]) if len(rp) else 0, rp.ctypes.data_as(C.POINTER(C.c_int32)),
                          col.ctypes.data_as(C.POINTER(C.c_int32)), val.ctypes.data_as(C.POINTER(C.c_double)))
    return s, (rp, col, val)


def min_bytes(n: int, nnz_u: int) -> int:
    """Algorithmic bytes of one SymmSpMV: Eq. 3 at alpha = 1/SymmNNZR:
    12 B per stored upper nonzero, 4 B per row pointer, x read once, y read+written once."""
    return 12 * nnz_u + 4 * (n + 1) + 24 * n


def flops(nnz_full: int) -> int:
    """2 flops per nonzero of the full symmetric matrix (north_star)."""
    return 2 * nnz_full


class Schedule:
    """race_schedule_t: BFS levels, permutation, level groups, tiles, colours, DAG."""

    def __init__(self, handle, n):
        self._h = handle
        self.n = n

    def __del__(self):
        if getattr(self, "_h", None):
            lib().race_schedule_destroy(self._h)
            self._h = None

    @property
    def stats(self) -> dict:
        st = _lib.RaceScheduleStats()
        check(lib().race_schedule_get_stats(self._h, C.byref(st)))
        return {f: getattr(st, f) for f, _ in _lib.RaceScheduleStats._fields_}

    def table(self, name: str) -> np.ndarray:
        ln = C.c_int64(0)
        check(lib().race_schedule_table(self._h, name.encode(), C.byref(ln), None))
        out = np.empty(ln.value, dtype=np.int32)
        if ln.value:
            check(lib().race_schedule_table(self._h, name.encode(), C.byref(ln), out.ctypes.data_as(C.POINTER(C.c_int32))))
        return out

    def permutation(self):
        perm = np.empty(self.n, dtype=np.int32)
        inv = np.empty(self.n, dtype=np.int32)
        if self.n:
            check(lib().race_schedule_permutation(self._h, perm.ctypes.data_as(C.POINTER(C.c_int32)),
                                                  inv.ctypes.data_as(C.POINTER(C.c_int32))))
        return perm, inv

    def partition(self, nranks: int):
        """Row bounds [nranks+1] and halo ends [nranks] of the multi-GPU split (R23)."""
        rb = np.empty(nranks + 1, dtype=np.int32)
        he = np.empty(nranks, dtype=np.int32)
        check(lib().race_schedule_partition(self._h, nranks, rb.ctypes.data_as(C.POINTER(C.c_int32)),
                                            he.ctypes.data_as(C.POINTER(C.c_int32))))
        return rb, he

    def permuted_matrix(self):
        nnz = self.stats["nnz"]
        rp = np.empty(self.n + 1, dtype=np.int32)
        col = np.empty(nnz, dtype=np.int32)
        val = np.empty(nnz, dtype=np.float64)
        check(lib().race_schedule_permuted_matrix(self._h, rp.ctypes.data_as(C.POINTER(C.c_int32)),
                                                  col.ctypes.data_as(C.POINTER(C.c_int32)),
                                                  val.ctypes.data_as(C.POINTER(C.c_double))))
        return rp, col, val


def default_config() -> dict:
    cfg = _lib.RaceConfig()
    lib().race_config_default(C.byref(cfg))
    d = {f: getattr(cfg, f) for f, _ in _lib.RaceConfig._fields_}
    d["eps"] = list(cfg.eps)
    return d


def build_schedule(U, **overrides) -> Schedule:
    """race_build_schedule(U, cfg): U has n, row_ptr, col, val (numpy, upper CRS)."""
    cfg = _lib.RaceConfig()
    lib().race_config_default(C.byref(cfg))
    for k, v in overrides.items():
        if k == "eps":
            for i, e in enumerate(v):
                cfg.eps[i] = e
            cfg.n_eps = len(v)
        elif hasattr(cfg, k):
            setattr(cfg, k, v)
        else:
            raise TypeError(f"unknown race_config field {k}")
    s, keep = _csr_struct(U)
    h = C.c_void_p()
    check(lib().race_build_schedule(C.byref(s), C.byref(cfg), C.byref(h)))
    return Schedule(h, int(U.n))


def halo_add(y, v, stream=None):
    """y += v on the device (C-ABI kernel), both contiguous CUDA float64 tensors."""
    check(lib().symmspmv_halo_add(C.c_void_p(_ptr(y)), C.c_void_p(_ptr(v)), int(v.numel()),
                                  C.c_void_p(_stream(stream))))


def bw_probe(mode: str = "load", nbytes: int = 4 << 30, reps: int = 5, device: int = 0, stream=None) -> float:
    """Measured HBM bandwidth in GB/s (symm_bw_probe, K5): "load" = load-only
    stream, "copy" = read + write (the roofline denominators of PAPER.md:440-456)."""
    g = C.c_double(0.0)
    check(lib().symm_bw_probe({"load": 0, "copy": 1}[mode], device, int(nbytes), int(reps),
                              C.c_void_p(_stream(stream)), C.byref(g)))
    return g.value


def _ptr(t):
    """Device pointer of a torch CUDA float64 tensor (or a raw int)."""
    if isinstance(t, int):
        return t
    import torch

    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise TypeError("expected a contiguous CUDA float64 tensor")
    return t.data_ptr()


def _stream(stream):
    if stream is None:
        import torch

        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class Plan:
    """symmspmv_plan_t: device-resident matrix + tables for one schedule."""

    def __init__(self, sched: Schedule, U=None, variant="auto", device: int = 0, vec_order="permuted",
                 vec_width: int = 0, build_all: bool = False, nranks: int = 1, rank: int = 0):
        o = _lib.SymmOptions()
        lib().symmspmv_options_default(C.byref(o))
        o.variant = VARIANTS[variant] if isinstance(variant, str) else int(variant)
        o.device = device
        o.vec_order = SYMM_ORDER_ORIGINAL if vec_order == "original" else SYMM_ORDER_PERMUTED
        o.vec_width = vec_width
        o.build_all = int(build_all)
        o.nranks = nranks
        o.rank = rank
        h = C.c_void_p()
        if U is not None:
            s, keep = _csr_struct(U)
            check(lib().symmspmv_plan(sched._h, C.byref(s), C.byref(o), C.byref(h)))
        else:
            check(lib().symmspmv_plan(sched._h, None, C.byref(o), C.byref(h)))
        self._h = h
        self.n = sched.n
        self.device = device

    def __del__(self):
        if getattr(self, "_h", None):
            lib().symmspmv_destroy(self._h)
            self._h = None

    def _check_dev(self, t, name):
        """x / y must be contiguous float64 tensors on the plan's device covering
        the plan's local rows (the kernels read / write that many elements)."""
        if isinstance(t, int):
            return t
        p = _ptr(t)
        if t.device.index != self.device:
            raise SymmError(-1, f"{name} is on cuda:{t.device.index}, the plan on cuda:{self.device}")
        b, e = self.local_range()
        if t.numel() < e - b:
            raise SymmError(-1, f"{name} has {t.numel()} elements, the plan needs {e - b}")
        return p

    def run(self, x, y, stream=None, variant=None):
        """y := A x (device tensors, asynchronous on `stream`)."""
        v = -1 if variant is None else (VARIANTS[variant] if isinstance(variant, str) else int(variant))
        check(lib().symmspmv_run_variant(self._h, v, C.c_void_p(self._check_dev(x, "x")),
                                         C.c_void_p(self._check_dev(y, "y")), C.c_void_p(_stream(stream))))

    def powers(self, x, Y, stream=None, variant=None):
        """Matrix powers: Y[k] := A^(k+1) x, k < Y.shape[0] (symmspmv_powers;
        Y a contiguous float64 device tensor of shape (npow, >= n))."""
        v = -1 if variant is None else (VARIANTS[variant] if isinstance(variant, str) else int(variant))
        if Y.dim() != 2 or Y.shape[1] < self.n or not Y.is_contiguous():
            raise SymmError(-1, f"Y must be a contiguous (npow, >= {self.n}) tensor")
        px = self._check_dev(x, "x")
        py = _ptr(Y) if Y.numel() else 0
        if Y.numel() and Y.device.index != self.device:
            raise SymmError(-1, f"Y is on cuda:{Y.device.index}, the plan on cuda:{self.device}")
        check(lib().symmspmv_powers(self._h, v, C.c_void_p(px), C.c_void_p(py), int(Y.shape[0]), int(Y.shape[1]),
                                    C.c_void_p(_stream(stream))))

    PARTS = {"all": 0, "interior": 1, "boundary": 2}

    def run_part(self, part, x, y, stream=None):
        """Multi-rank halo overlap (symmspmv_run_part): "interior" zeroes y and
        runs the tiles that touch only own rows, "boundary" the tiles that
        touch halo rows (after the x halo has arrived)."""
        pt = self.PARTS[part] if isinstance(part, str) else int(part)
        check(lib().symmspmv_run_part(self._h, pt, C.c_void_p(self._check_dev(x, "x")),
                                      C.c_void_p(self._check_dev(y, "y")), C.c_void_p(_stream(stream))))

    def parts(self) -> dict:
        """Tiles / stored nonzeros of the interior and boundary parts."""
        ti, tb, ni, nb = C.c_int32(0), C.c_int32(0), C.c_int64(0), C.c_int64(0)
        check(lib().symmspmv_plan_parts(self._h, C.byref(ti), C.byref(tb), C.byref(ni), C.byref(nb)))
        return {"interior_tiles": ti.value, "boundary_tiles": tb.value, "interior_nnz": ni.value,
                "boundary_nnz": nb.value}

    def run_host(self, x: np.ndarray, y: np.ndarray, stream=None):
        """End to end: HOST fp64 vectors in ORIGINAL order (pinned recommended)."""
        for name, a in (("x", x), ("y", y)):
            if not isinstance(a, np.ndarray):
                raise TypeError(f"{name} must be a numpy array")
            if a.dtype != np.float64 or not a.flags.c_contiguous or a.size < self.n:
                raise SymmError(-1, f"{name} must be a C-contiguous float64 array of >= {self.n} elements")
        if not y.flags.writeable:
            raise SymmError(-1, "y is read-only")
        check(lib().symmspmv_run_host(self._h, C.c_void_p(x.ctypes.data), C.c_void_p(y.ctypes.data),
                                      C.c_void_p(_stream(stream))))

    def local_range(self):
        """(row_begin, local_end): the rows x / y passed to run() cover."""
        b, e = C.c_int32(0), C.c_int32(0)
        check(lib().symmspmv_plan_local(self._h, C.byref(b), C.byref(e)))
        return b.value, e.value

    def own_rows(self):
        b, e = C.c_int32(0), C.c_int32(0)
        check(lib().symmspmv_plan_rows(self._h, C.byref(b), C.byref(e)))
        return b.value, e.value

    @property
    def last_launches(self) -> int:
        return int(lib().symmspmv_last_launches(self._h))

    def info(self) -> dict:
        out = (C.c_int32 * 8)()
        m = lib().symmspmv_plan_info(self._h, out, 8)
        keys = ["variant", "vec", "tiled_grid", "tiled_stages", "block_cap", "window_cap", "nnz_cap", "tiled_smem"]
        return {keys[i]: int(out[i]) for i in range(max(m, 0))}

    def bytes(self):
        d, m = C.c_int64(0), C.c_int64(0)
        check(lib().symmspmv_plan_bytes(self._h, C.byref(d), C.byref(m)))
        return d.value, m.value


class Sweep:
    """symm_sweep_t (NEXT-4): Gauss-Seidel ("gs", distance-1) or Kaczmarz
    ("kacz", distance-2) sweeps phase by phase on the schedule's level groups,
    rows coloured inside every group (include/symmspmv.h)."""

    KINDS = {"gs": 1, "kacz": 2}

    def __init__(self, sched: Schedule, kind: str = "kacz", device: int = 0):
        h = C.c_void_p()
        check(lib().symm_sweep_plan(sched._h, self.KINDS[kind], device, C.byref(h)))
        self._h = h
        self.n = sched.n
        self.kind = kind

    def __del__(self):
        if getattr(self, "_h", None):
            lib().symm_sweep_destroy(self._h)
            self._h = None

    def run(self, x, b, symmetric: bool = True, stream=None):
        """x := sweep(x) (device tensors in the permuted order, asynchronous)."""
        check(lib().symm_sweep_run(self._h, C.c_void_p(_ptr(x)), C.c_void_p(_ptr(b)), int(symmetric),
                                   C.c_void_p(_stream(stream))))

    def order(self):
        """(rows in execution order (permuted ids), phase_ptr)."""
        npz = C.c_int32(0)
        check(lib().symm_sweep_order(self._h, None, None, C.byref(npz)))
        rows = np.zeros(self.n, dtype=np.int32)
        ptr = np.zeros(npz.value + 1, dtype=np.int32)
        check(lib().symm_sweep_order(self._h, rows.ctypes.data, ptr.ctypes.data, C.byref(npz)))
        return rows, ptr
