"""Seeded synthetic inputs shared by tests (oracle side) and bench (product side).

This package holds NO SymmSpMV/RACE arithmetic: it builds upper-triangular CRS
matrices (int32 indices, fp64 values, diagonal first, ascending columns) and
input vectors from a seed.  The heavy builders live in ``symmgen.cpp``
(``libsymmgen.so``); small structural test graphs are built here with numpy.

The five named configs follow BASELINE.json ``configs`` (DESIGN.md "Input
recipe" gives the readings taken where the config text is silent).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libsymmgen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make` (or __graft_entry__.build()) first")
        L = C.CDLL(path)
        vp = C.c_void_p
        for name, args in {
            "gen_lap2d": [C.c_int32],
            "gen_lap3d": [C.c_int32, C.c_uint64, C.c_int32],
            "gen_spin": [C.c_int32, C.c_uint64],
            "gen_st27": [C.c_int32, C.c_uint64, C.c_int32],
            "gen_knn": [C.c_int32, C.c_int32, C.c_uint64],
            "gen_from_edges": [C.c_int32, C.c_int64, vp, vp, vp, vp, vp],
        }.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = vp
        L.gen_n.argtypes = [vp]
        L.gen_n.restype = C.c_int32
        L.gen_nnz.argtypes = [vp]
        L.gen_nnz.restype = C.c_int64
        for name, ct in (("gen_row_ptr", C.c_int32), ("gen_col", C.c_int32), ("gen_val", C.c_double)):
            f = getattr(L, name)
            f.argtypes = [vp]
            f.restype = C.POINTER(ct)
        L.gen_free.argtypes = [vp]
        L.gen_free.restype = None
        L.gen_vector_uniform.argtypes = [C.c_int64, C.c_uint64, C.c_double, C.c_double, vp]
        L.gen_vector_uniform.restype = None
        L.gen_vector_sinsin.argtypes = [C.c_int32, vp]
        L.gen_vector_sinsin.restype = None
        L.gen_num_threads.restype = C.c_int
        _LIB = L
    return _LIB


class _Handle:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        if self.h:
            _lib().gen_free(self.h)
            self.h = None


@dataclass
class UpperCSR:
    """Upper triangle U of a symmetric A (A = U + U^T - diag(U)), 0-based CRS."""

    n: int
    row_ptr: np.ndarray  # int32[n+1]
    col: np.ndarray  # int32[nnz]
    val: np.ndarray  # float64[nnz]
    name: str = ""
    _keep: object = field(default=None, repr=False)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1]) if self.n > 0 else 0

    def nnz_full(self) -> int:
        """Nonzeros of A = U + U^T - diag: 2*nnz_u - (#stored diagonal entries)."""
        rows = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.row_ptr))
        ndiag = int(np.count_nonzero(self.col == rows))
        return 2 * self.nnz - ndiag


def _wrap(h, name: str) -> UpperCSR:
    if not h:
        raise MemoryError(f"generator {name} failed (size overflow or OOM)")
    L = _lib()
    keep = _Handle(h)
    n = L.gen_n(h)
    nnz = L.gen_nnz(h)
    rp = np.ctypeslib.as_array(L.gen_row_ptr(h), shape=(n + 1,))
    col = np.ctypeslib.as_array(L.gen_col(h), shape=(max(nnz, 1),))[:nnz]
    val = np.ctypeslib.as_array(L.gen_val(h), shape=(max(nnz, 1),))[:nnz]
    return UpperCSR(n=n, row_ptr=rp, col=col, val=val, name=name, _keep=keep)


def lap2d(N: int) -> UpperCSR:
    return _wrap(_lib().gen_lap2d(N), f"lap2d_{N}")


def lap3d(N: int, seed: int = 5, perturb: bool = True) -> UpperCSR:
    return _wrap(_lib().gen_lap3d(N, seed, int(perturb)), f"lap3d_{N}")


def spin(L: int, seed: int = 4) -> UpperCSR:
    return _wrap(_lib().gen_spin(L, seed), f"spin_{L}")


def st27(N: int, seed: int = 2, shuffle: bool = True) -> UpperCSR:
    return _wrap(_lib().gen_st27(N, seed, int(shuffle)), f"st27_{N}")


def knn(npts: int, k: int = 20, seed: int = 3) -> UpperCSR:
    return _wrap(_lib().gen_knn(npts, k, seed), f"knn_{npts}_{k}")


def from_edges(n: int, u, v, w=None, diag=None, has_diag=None, name="edges") -> UpperCSR:
    """Upper CRS of the symmetric matrix with the given undirected edges (listed once)."""
    u = np.ascontiguousarray(u, dtype=np.int32)
    v = np.ascontiguousarray(v, dtype=np.int32)
    m = len(u)
    w = np.ascontiguousarray(np.ones(m) if w is None else w, dtype=np.float64)
    d = np.ascontiguousarray(np.ones(n) if diag is None else diag, dtype=np.float64)
    hd = np.ascontiguousarray(np.ones(n, dtype=np.int8) if has_diag is None else has_diag, dtype=np.int8)
    if m and (np.any(u == v) or u.min() < 0 or v.min() < 0 or max(u.max(), v.max()) >= n):
        raise ValueError("edges must join distinct in-range vertices")
    h = _lib().gen_from_edges(n, m, u.ctypes.data, v.ctypes.data, w.ctypes.data, d.ctypes.data, hd.ctypes.data)
    return _wrap(h, name)


def random_symmetric(n: int, avg_deg: float, seed: int, diag_frac: float = 1.0, name=None) -> UpperCSR:
    """Random simple graph (Erdos-Renyi-like, ~avg_deg neighbours/vertex), values U(-1,1)."""
    rng = np.random.default_rng(seed)
    m = int(round(n * avg_deg / 2))
    if n < 2:
        m = 0
    a = rng.integers(0, max(n, 1), size=m)
    b = rng.integers(0, max(n, 1), size=m)
    keep = a != b
    a, b = a[keep], b[keep]
    lo, hi = np.minimum(a, b), np.maximum(a, b)
    key = np.unique(lo.astype(np.int64) * n + hi)
    lo, hi = (key // max(n, 1)).astype(np.int32), (key % max(n, 1)).astype(np.int32)
    w = rng.uniform(-1, 1, size=len(lo))
    d = rng.uniform(-1, 1, size=n) + 4.0
    hd = (rng.uniform(size=n) < diag_frac).astype(np.int8)
    return from_edges(n, lo, hi, w, d, hd, name or f"rand_{n}_{avg_deg}_{seed}")


def banded_random(n: int, bw: int, avg_deg: float, seed: int) -> UpperCSR:
    """Random symmetric graph whose edges join vertices at most ``bw`` apart."""
    rng = np.random.default_rng(seed)
    m = int(round(n * avg_deg / 2))
    a = rng.integers(0, n, size=m)
    off = rng.integers(1, bw + 1, size=m)
    b = a + off
    keep = b < n
    a, b = a[keep], b[keep]
    key = np.unique(a.astype(np.int64) * n + b)
    lo, hi = (key // n).astype(np.int32), (key % n).astype(np.int32)
    w = rng.uniform(-1, 1, size=len(lo))
    d = rng.uniform(3, 5, size=n)
    return from_edges(n, lo, hi, w, d, None, f"band_{n}_{bw}_{seed}")


def path(n: int) -> UpperCSR:
    i = np.arange(n - 1, dtype=np.int32)
    return from_edges(n, i, i + 1, name=f"path_{n}")


def vector_uniform(n: int, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    if n:
        _lib().gen_vector_uniform(n, seed, lo, hi, out.ctypes.data)
    return out


def vector_sinsin(N: int) -> np.ndarray:
    out = np.empty(N * N, dtype=np.float64)
    _lib().gen_vector_sinsin(N, out.ctypes.data)
    return out


def num_threads() -> int:
    return int(_lib().gen_num_threads())


# --- the five BASELINE.json configs (index = position in BASELINE.json configs) ---
CONFIGS = {
    "lap2d_64": dict(index=0, build=lambda: lap2d(64), x_seed=101),
    "st27_128": dict(index=1, build=lambda: st27(128, 2, True), x_seed=102),
    "fem_knn_4M": dict(index=2, build=lambda: knn(4_000_000, 20, 3), x_seed=103),
    "spin_22": dict(index=3, build=lambda: spin(22, 4), x_seed=104),
    "lap3d_512": dict(index=4, build=lambda: lap3d(512, 5, True), x_seed=105),
}

# Reduced-size members of the same families (same generators, same seeds) for
# parity tests the oracle finishes in seconds.
SMALL_CONFIGS = {
    "lap2d_64": dict(build=lambda: lap2d(64), x_seed=101),
    "st27_24": dict(build=lambda: st27(24, 2, True), x_seed=102),
    "fem_knn_30k": dict(build=lambda: knn(30_000, 20, 3), x_seed=103),
    "spin_14": dict(build=lambda: spin(14, 4), x_seed=104),
    "lap3d_40": dict(build=lambda: lap3d(40, 5, True), x_seed=105),
}


# Mid-size members used for profiling and scaling studies (not BASELINE configs).
EXTRA_CONFIGS = {
    "lap3d_256": dict(build=lambda: lap3d(256, 5, True), x_seed=105),
    "fem_knn_1M": dict(build=lambda: knn(1_000_000, 20, 3), x_seed=103),
}


def make_config(name: str):
    spec = CONFIGS.get(name) or SMALL_CONFIGS.get(name) or EXTRA_CONFIGS[name]
    U = spec["build"]()
    U.name = name
    return U, vector_uniform(U.n, spec["x_seed"])
