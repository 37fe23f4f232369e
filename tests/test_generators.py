"""Pins of the seeded input generators (gen/, shared by tests and bench; they
hold none of the method's arithmetic).  SURVEY §8(c) "Generators" row and
DESIGN.md §4 (readings R19-R22):

* closed-form nonzero counts of the stencil / spin families at the full
  BASELINE.json sizes: 5n - 4N (2-D 5-pt), (3N-2)^3 (27-pt), 22n (spin),
  7n - 6N^2 (7-pt); every row stores its diagonal, so nnz_u = (nnz_full + n)/2;
* value symmetry: configs 2 and 3 set diag_i = sum_j |a_ij| + 1 over the FULL
  row (R20), which holds only if the mirrored copies of every edge value agree
  (values keyed per unordered pair, R22) -> strict diagonal dominance;
* spin: i couples to i XOR (3 << b), b = 0..20: a Cayley graph of (Z_2)^22 with
  21 independent generators, i.e. two cosets, each a 21-cube -> exactly two
  components of 2^21 rows and BFS level sizes C(21, d) from any root;
* determinism: bitwise identical matrices with 1 and 8 OpenMP threads.
"""
import hashlib
import json
import math
import os
import subprocess
import sys

import numpy as np
import pytest

import gen
import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rows(U):
    return np.repeat(np.arange(U.n, dtype=np.int64), np.diff(U.row_ptr))


def _diag_count(U):
    return int(np.count_nonzero(U.col == _rows(U)))


@pytest.mark.parametrize("name,N,formula", [
    ("lap2d_64", 64, lambda n, N: 5 * n - 4 * N),
    ("st27_128", 128, lambda n, N: (3 * N - 2) ** 3),
    ("spin_22", 22, lambda n, N: 22 * n),
    ("lap3d_512", 512, lambda n, N: 7 * n - 6 * N * N),
])
def test_closed_form_nnz_full_size(name, N, formula):
    spec = gen.CONFIGS[name]
    U = spec["build"]()
    n = U.n
    expect_n = {"lap2d_64": N * N, "st27_128": N ** 3, "spin_22": 2 ** N, "lap3d_512": N ** 3}[name]
    assert n == expect_n
    nd = _diag_count(U)
    assert nd == n  # every row stores its diagonal
    nnz_full = 2 * U.nnz - nd
    assert nnz_full == formula(n, N)
    assert U.nnz == (nnz_full + n) // 2
    # upper CRS: col >= row, strictly ascending per row
    rows = _rows(U)
    assert np.all(U.col >= rows)
    d = np.diff(U.col.astype(np.int64))
    same_row = rows[1:] == rows[:-1]
    assert np.all(d[same_row] > 0)


def test_printed_sizes():
    """The sizes SURVEY §8(a) prints."""
    assert 5 * 4096 - 4 * 64 == 20224
    assert (3 * 128 - 2) ** 3 == 55_742_968
    assert 22 * 2 ** 22 == 92_274_688
    assert 7 * 512 ** 3 - 6 * 512 ** 2 == 937_951_232
    assert (937_951_232 + 512 ** 3) // 2 == 536_084_480


def _full_row_abs_sum(U):
    """sum_{j != i} |A_ij| over the full symmetric row (upper entries of row i
    plus the mirrored entries stored in earlier rows)."""
    rows = _rows(U)
    off = U.col != rows
    a = np.abs(U.val[off])
    s = np.zeros(U.n)
    np.add.at(s, rows[off], a)
    np.add.at(s, U.col[off], a)
    return s, U.val[~off], rows[~off]


@pytest.mark.parametrize("name", ["st27_128", "fem_knn_4M"])
def test_diagonal_dominance_full_size(name):
    """Configs 2 and 3: diag = sum |a| + 1 (R20) -> strictly diagonally dominant.
    The equality is checked over the FULL row, so it also pins value symmetry."""
    U, _ = gen.make_config(name)
    s, dv, dr = _full_row_abs_sum(U)
    assert len(dr) == U.n
    assert np.all(dv > s)  # strict dominance
    assert np.max(np.abs(dv - (s[dr] + 1.0)) / (s[dr] + 1.0)) < 1e-13
    off = U.col != _rows(U)
    if name == "st27_128":
        assert np.all((U.val[off] >= -1.0) & (U.val[off] <= 0.0))  # U(-1, 0)
    else:
        assert np.all((U.val[off] >= -1.0) & (U.val[off] <= 1.0))  # U(-1, 1)
        nnzr = (2 * U.nnz - U.n) / U.n
        assert 22.0 < nnzr < 25.0  # k = 20 union-symmetrised (R19): ~23.3 per row


def test_spin_two_components_binomial_levels_full_size():
    U, _ = gen.make_config("spin_22")
    n, L = U.n, 22
    rows = _rows(U)
    off = U.col != rows
    # every off-diagonal entry is i XOR (3 << b), value 0.5
    x = rows[off] ^ U.col[off].astype(np.int64)
    allowed = np.array([3 << b for b in range(L - 1)], dtype=np.int64)
    assert np.all(np.isin(x, allowed))
    assert np.all(U.val[off] == 0.5)
    assert 2 * int(off.sum()) == (L - 1) * n  # 21 neighbours per row
    gp, ga = oracle.graph(U)
    # BFS from row 0; the second island starts two levels further (R10)
    dist, tl = oracle.bfs_levels(gp, ga, [0])
    sizes = np.bincount(dist, minlength=tl)
    binom = np.array([math.comb(L - 1, d) for d in range(L)])
    assert tl == 2 * L + 1
    assert np.array_equal(sizes[:L], binom)
    assert sizes[L] == 0  # empty separator level
    assert np.array_equal(sizes[L + 1:], binom)
    # the two components are the two cosets of the generated subspace: every
    # generator 3 << b flips two bits, so the popcount parity is invariant and
    # row 0's component is exactly the even-popcount rows
    pc = np.array([bin(i).count("1") & 1 for i in range(0, n, 4097)])
    d_s = dist[::4097]
    assert np.all((d_s <= L - 1) == (pc == 0))


_HASH_SCRIPT = r"""
import hashlib, json, sys
sys.path.insert(0, {root!r})
import gen
out = {{}}
for name, mk in (("st27", lambda: gen.st27(40, 2, True)), ("knn", lambda: gen.knn(60000, 20, 3)),
                 ("spin", lambda: gen.spin(16, 4)), ("lap3d", lambda: gen.lap3d(48, 5, True)),
                 ("x", None)):
    h = hashlib.sha256()
    if mk is None:
        h.update(gen.vector_uniform(100000, 103).tobytes())
    else:
        U = mk()
        for a in (U.row_ptr, U.col, U.val):
            h.update(a.tobytes())
    out[name] = h.hexdigest()
out["threads"] = gen.num_threads()
print(json.dumps(out))
"""


def _hashes(nthreads):
    env = dict(os.environ, OMP_NUM_THREADS=str(nthreads))
    r = subprocess.run([sys.executable, "-c", _HASH_SCRIPT.format(root=ROOT)], capture_output=True, text=True,
                       env=env, timeout=300)
    assert r.returncode == 0, r.stderr
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_bitwise_identical_across_thread_counts():
    h1, h8 = _hashes(1), _hashes(8)
    assert h1.pop("threads") == 1 and h8.pop("threads") == 8
    assert h1 == h8
