"""ORACLE — TEST INFRASTRUCTURE ONLY.

Plain CPU reference for the SymmSpMV hot path of arXiv 1907.06487 (RACE).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It
shares no code with the product (``paper_1907_06487_b200``) and never imports
it.

* ``liboracle.so`` (``oracle.c``): Alg. 2 SymmSpMV, Alg. 1 SpMV, mirror,
  dense matvec, Alg. 3 BFS levels (+ island rule), brute-force distance-k and
  write-conflict checks.
* ``matrix_powers``: A^k x, k = 1..p, by repeated Alg. 2 (NEXT-4).
* ``race.py``: §4.4.3 epsilon level aggregation, Alg. 4 load balancing, §5
  effective row count / eta — pure Python, step by step in the paper's order.
* ``perfmodel.py``: Eq. 1-4 and the alpha inversion of §3.3.

Parity status of every function is listed in DESIGN.md ("Oracle pins").
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make` (or __graft_entry__.build()) first")
        L = C.CDLL(path)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        L.oracle_symmspmv.argtypes = [i32, vp, vp, vp, vp, vp]
        L.oracle_symmspmv.restype = None
        L.oracle_symmspmv_ld.argtypes = [i32, vp, vp, vp, vp, vp]
        L.oracle_symmspmv_ld.restype = None
        L.oracle_symmspmv_omp.argtypes = [i32, vp, vp, vp, vp, vp, i32]
        L.oracle_symmspmv_omp.restype = i32
        L.oracle_gs_sweep.argtypes = [i32, vp, vp, vp, vp, vp, vp, i64]
        L.oracle_gs_sweep.restype = None
        L.oracle_kacz_sweep.argtypes = [i32, vp, vp, vp, vp, vp, vp, i64]
        L.oracle_kacz_sweep.restype = None
        L.oracle_mirror.argtypes = [i32, vp, vp, vp, vp, vp, vp]
        L.oracle_mirror.restype = i64
        L.oracle_spmv.argtypes = [i32, vp, vp, vp, vp, vp]
        L.oracle_spmv.restype = None
        L.oracle_dense_matvec.argtypes = [i32, vp, vp, vp]
        L.oracle_dense_matvec.restype = None
        L.oracle_bfs_levels.argtypes = [i32, vp, vp, i32, vp, vp]
        L.oracle_bfs_levels.restype = i32
        L.oracle_distk_violations.argtypes = [i32, vp, vp, i32, vp]
        L.oracle_distk_violations.restype = i64
        L.oracle_write_conflicts.argtypes = [i32, vp, vp, vp]
        L.oracle_write_conflicts.restype = i64
        _LIB = L
    return _LIB


def _p(a):
    return a.ctypes.data


def _csr(U):
    return (np.ascontiguousarray(U.row_ptr, dtype=np.int32), np.ascontiguousarray(U.col, dtype=np.int32),
            np.ascontiguousarray(U.val, dtype=np.float64))


def symmspmv(U, x) -> np.ndarray:
    """y = A x from the upper triangle U via Alg. 2, fp64, serial."""
    rp, col, val = _csr(U)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(U.n, dtype=np.float64)
    _lib().oracle_symmspmv(U.n, _p(rp), _p(col), _p(val), _p(x), _p(y))
    return y


def symmspmv_omp(U, x, nthreads: int = 0):
    """Alg. 2 with thread-private target arrays, OpenMP;
    returns (y, threads used).  Host-core baseline for bench.py only."""
    rp, col, val = _csr(U)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(U.n, dtype=np.float64)
    nt = _lib().oracle_symmspmv_omp(U.n, _p(rp), _p(col), _p(val), _p(x), _p(y), int(nthreads))
    if nt < 0:
        raise MemoryError("oracle_symmspmv_omp: allocation failed")
    return y, nt


def symmspmv_ld(U, x) -> np.ndarray:
    """Alg. 2 with long-double accumulation (diagnostic reference grade)."""
    rp, col, val = _csr(U)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(U.n, dtype=np.longdouble)
    _lib().oracle_symmspmv_ld(U.n, _p(rp), _p(col), _p(val), _p(x), _p(y))
    return y


def mirror(U):
    """Full CRS of A = U + U^T - diag(U): (row_ptr, col, val), sorted rows."""
    rp, col, val = _csr(U)
    frp = np.empty(U.n + 1, dtype=np.int32)
    nnz = _lib().oracle_mirror(U.n, _p(rp), _p(col), _p(val), _p(frp), None, None)
    fcol = np.empty(max(nnz, 1), dtype=np.int32)
    fval = np.empty(max(nnz, 1), dtype=np.float64)
    _lib().oracle_mirror(U.n, _p(rp), _p(col), _p(val), _p(frp), _p(fcol), _p(fval))
    return frp, fcol[:nnz], fval[:nnz]


def spmv(rp, col, val, x) -> np.ndarray:
    """Alg. 1 on a full CRS matrix."""
    rp = np.ascontiguousarray(rp, dtype=np.int32)
    col = np.ascontiguousarray(col, dtype=np.int32)
    val = np.ascontiguousarray(val, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    n = len(rp) - 1
    y = np.empty(n, dtype=np.float64)
    _lib().oracle_spmv(n, _p(rp), _p(col), _p(val), _p(x), _p(y))
    return y


def matrix_powers(U, x, npow: int) -> np.ndarray:
    """Matrix powers [A x, A^2 x, ..., A^npow x] (rows of the result), by the
    plain definition y_0 = x, y_k = A y_{k-1}, each step one Alg. 2 SymmSpMV
    (PAPER.md:730-745).  The paper names "in-place matrix powers and
    polynomials" as the level-based formulation's next kernels
    (§8 Conclusion); it gives no algorithm, so the oracle
    is the definition itself."""
    Y = np.empty((max(int(npow), 0), U.n), dtype=np.float64)
    y = np.ascontiguousarray(x, dtype=np.float64)
    for k in range(int(npow)):
        y = symmspmv(U, y)
        Y[k] = y
    return Y


def sweep(kind: str, U, b, x0, order, symmetric: bool = False) -> np.ndarray:
    """One serial Gauss-Seidel ("gs") or Kaczmarz ("kacz") sweep over the rows
    in `order` (then in reverse if symmetric) on the full matrix of U
    (readings R32-R33); returns the new x."""
    rp, col, val = mirror(U)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.array(x0, dtype=np.float64, copy=True)
    f = _lib().oracle_gs_sweep if kind == "gs" else _lib().oracle_kacz_sweep
    for o in ([order, order[::-1]] if symmetric else [order]):
        o = np.ascontiguousarray(o, dtype=np.int32)
        f(U.n, _p(rp), _p(col), _p(val), _p(b), _p(x), _p(o), len(o))
    return x


def dense_matvec(Ad, x) -> np.ndarray:
    Ad = np.ascontiguousarray(Ad, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(Ad.shape[0], dtype=np.float64)
    _lib().oracle_dense_matvec(Ad.shape[0], _p(Ad), _p(x), _p(y))
    return y


def to_dense(U) -> np.ndarray:
    """Dense A from U by the definition A_ij = A_ji = U_ij (i <= j)."""
    A = np.zeros((U.n, U.n))
    for r in range(U.n):
        for idx in range(U.row_ptr[r], U.row_ptr[r + 1]):
            c = U.col[idx]
            A[r, c] = U.val[idx]
            A[c, r] = U.val[idx]
    return A


def graph(U):
    """Full symmetric adjacency (no self loops) of the pattern of A."""
    frp, fcol, _ = mirror(U)
    rows = np.repeat(np.arange(U.n, dtype=np.int32), np.diff(frp))
    keep = fcol != rows
    gp = np.zeros(U.n + 1, dtype=np.int32)
    np.cumsum(np.bincount(rows[keep], minlength=U.n), out=gp[1:])
    return gp, np.ascontiguousarray(fcol[keep], dtype=np.int32)


def bfs_levels(g_ptr, g_adj, roots=()) -> tuple[np.ndarray, int]:
    """Alg. 3 + island rule: (dist, totalLvl)."""
    g_ptr = np.ascontiguousarray(g_ptr, dtype=np.int32)
    g_adj = np.ascontiguousarray(g_adj, dtype=np.int32)
    n = len(g_ptr) - 1
    r = np.ascontiguousarray(np.asarray(roots, dtype=np.int32))
    dist = np.empty(n, dtype=np.int32)
    tl = _lib().oracle_bfs_levels(n, _p(g_ptr), _p(g_adj) if len(g_adj) else None, len(r),
                                  _p(r) if len(r) else None, _p(dist))
    return dist, int(tl)


def distk_violations(g_ptr, g_adj, k: int, cls) -> int:
    """Brute-force Eq. 6 relation: ordered same-class pairs within distance k."""
    g_ptr = np.ascontiguousarray(g_ptr, dtype=np.int32)
    g_adj = np.ascontiguousarray(g_adj, dtype=np.int32)
    cls = np.ascontiguousarray(cls, dtype=np.int32)
    return int(_lib().oracle_distk_violations(len(g_ptr) - 1, _p(g_ptr), _p(g_adj) if len(g_adj) else None,
                                              k, _p(cls)))


def write_conflicts(U, cls) -> int:
    """Pairs of same-class rows of Alg. 2 whose write sets {r} ∪ cols(r) intersect."""
    rp, col, _ = _csr(U)
    cls = np.ascontiguousarray(cls, dtype=np.int32)
    return int(_lib().oracle_write_conflicts(U.n, _p(rp), _p(col), _p(cls)))


def conflicting_row_pairs(U):
    """All unordered row pairs (r, s), r < s, whose Alg. 2 write sets intersect.

    Definition: row r writes b[r] and b[c] for each stored
    c > r.  Plain enumeration by target: every pair of writers of one target.
    """
    writers = [[] for _ in range(U.n)]
    for r in range(U.n):
        writers[r].append(r)
        for idx in range(U.row_ptr[r], U.row_ptr[r + 1]):
            c = int(U.col[idx])
            if c != r:
                writers[c].append(r)
    pairs = set()
    for ws in writers:
        ws = sorted(set(ws))
        for i in range(len(ws)):
            for j in range(i + 1, len(ws)):
                pairs.add((ws[i], ws[j]))
    return pairs
