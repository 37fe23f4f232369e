"""Host-side tests of the C-ABI library (no GPU): exports, input validation,
BFS levels / permutation vs the oracle, RACE aggregation + Alg. 4 parity vs the
Python oracle, and brute-force validity of the conflict-free schedule."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import gen
import oracle
import paper_1907_06487_b200 as P
from oracle import race
from paper_1907_06487_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "symmspmv.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    names = set(re.findall(r"^\s*(?:const\s+)?(?:int|void|char)\s*\*?\s*(\w+)\s*\(", hdr, flags=re.M))
    assert len(names) >= 15
    L = C.CDLL(_lib.LIB_PATH)
    for name in names:
        assert hasattr(L, name), name
    assert names == set(_lib.EXPORTS)


def _bad(U, code, **kw):
    with pytest.raises(P.SymmError) as e:
        P.build_schedule(U, **kw)
    assert e.value.code == code
    return str(e.value)


def test_input_validation_errors():
    class M:
        pass

    m = M()
    m.n, m.row_ptr, m.col, m.val = 3, np.array([0, 2, 3, 4]), np.array([0, 1, 0, 2]), np.ones(4)
    msg = _bad(m, -2)  # row 1 stores col 0 < row
    assert "row 1" in msg
    m.col = np.array([1, 0, 1, 2])
    _bad(m, -3)  # row 0 columns not ascending
    m.col = np.array([0, 0, 1, 2])
    _bad(m, -3)  # duplicate
    m.col = np.array([0, 1, 1, 5])
    _bad(m, -2)  # col >= n
    m.row_ptr = np.array([0, 2, 1, 4])
    m.col = np.array([0, 1, 1, 2])
    _bad(m, -1)  # row_ptr decreasing
    U = gen.lap2d(4)
    _bad(U, -11, k=1)  # SymmSpMV needs distance 2
    _bad(U, -1, max_tile_window=10)


def _levels_from_dist(dist):
    return np.bincount(dist, minlength=int(dist.max()) + 1)


GRAPHS = [
    ("lap2d_17", lambda: gen.lap2d(17)),
    ("st27_9", lambda: gen.st27(9, 2, True)),
    ("spin_9", lambda: gen.spin(9, 4)),
    ("knn_800", lambda: gen.knn(800, 8, 3)),
    ("lap3d_9", lambda: gen.lap3d(9, 5, True)),
    ("rand_300", lambda: gen.random_symmetric(300, 3.0, 4, diag_frac=0.7)),
    ("rand_islands", lambda: gen.random_symmetric(400, 1.2, 5)),
    ("band_500", lambda: gen.banded_random(500, 12, 6.0, 6)),
]


@pytest.mark.parametrize("name,mk", GRAPHS)
def test_bfs_levels_match_oracle(name, mk):
    U = mk()
    s = P.build_schedule(U)
    roots = s.table("roots")
    dist = s.table("dist")
    gp, ga = oracle.graph(U)
    d_or, tl = oracle.bfs_levels(gp, ga, roots)
    assert np.array_equal(dist, d_or)  # Eq. 5 levels are unique given the roots
    lp = s.table("level_ptr")
    assert len(lp) == tl + 1 and s.stats["total_levels"] == tl
    assert np.array_equal(np.diff(lp), _levels_from_dist(d_or))
    perm, inv = s.permutation()
    assert np.array_equal(np.sort(perm), np.arange(U.n)) and np.array_equal(perm[inv], np.arange(U.n))
    # levels contiguous and ascending in the permuted order
    assert np.all(np.diff(dist[inv]) >= 0)
    assert s.stats["n_components"] == len(roots)


@pytest.mark.parametrize("name,mk", GRAPHS)
def test_permuted_matrix_is_PAPt(name, mk):
    U = mk()
    s = P.build_schedule(U)
    perm, inv = s.permutation()
    rp, col, val = s.permuted_matrix()
    Up = gen.UpperCSR(U.n, rp, col, val)
    x = gen.vector_uniform(U.n, 3)
    y = oracle.symmspmv(U, x)
    yp = oracle.symmspmv(Up, x[inv])  # (P A P^T)(P x) = P (A x)
    assert np.max(np.abs(yp - y[inv])) <= 1e-13 * max(1.0, np.max(np.abs(y)))
    assert np.all(np.diff(rp) >= 0)
    rows = np.repeat(np.arange(U.n), np.diff(rp))
    assert np.all(col >= rows)


@pytest.mark.parametrize("name,mk", GRAPHS)
@pytest.mark.parametrize("tile_work", [64, 512, 16384])
def test_race_aggregation_and_alg4_match_oracle(name, mk, tile_work):
    """eps windows (§4.4.3) and Alg. 4 groups (§4.3) bit-identical to the oracle."""
    U = mk()
    s = P.build_schedule(U, tile_work=tile_work)
    lp = s.table("level_ptr")
    rp, _, _ = s.permuted_matrix()
    row_work = np.diff(rp).astype(np.int64) + 2
    lw = [int(row_work[lp[i]:lp[i + 1]].sum()) for i in range(len(lp) - 1)]
    W = max(1, -(-sum(lw) // tile_work))
    win = race.eps_aggregate(lw, W, 2, 0.8)
    got = s.table("window_levels").reshape(-1, 3)
    assert [tuple(map(int, r)) for r in got] == win
    T, wk = [win[0][0]], []
    for f, l, b in win:
        T += [race.split_window(lw, f, l, 2), l]
        wk += [b, b]
    T, _ = race.alg4_balance(T, wk, lw, kmin=2)
    assert list(s.table("group_lvl")) == T
    assert list(s.table("group_workers")) == wk


def _check_schedule_bruteforce(U, s):
    """Every pair of rows whose Alg. 2 write sets intersect must be ordered:
    same tile -> different intra-tile colours; different tiles -> a DAG edge
    between the tiles, and different phases."""
    perm, inv = s.permutation()
    tp = s.table("tile_ptr")
    tile_of = np.repeat(np.arange(len(tp) - 1), np.diff(tp))
    sub = s.table("row_subcolor")
    phase = s.table("tile_phase")
    dp, dpred = s.table("dag_ptr"), s.table("dag_pred")
    edges = set()
    for t in range(len(tp) - 1):
        for u in dpred[dp[t]:dp[t + 1]]:
            edges.add((int(u), t))
            assert phase[u] < phase[t]
    rp, col, val = s.permuted_matrix()
    Up = gen.UpperCSR(U.n, rp, col, val)
    for (a, b) in oracle.conflicting_row_pairs(Up):
        ta, tb = tile_of[a], tile_of[b]
        if ta == tb:
            assert sub[a] != sub[b], (a, b)
        else:
            assert phase[ta] != phase[tb]
            assert (ta, tb) in edges or (tb, ta) in edges, (a, b, ta, tb)
    # the claim order is a topological order of the DAG
    order = s.table("tile_order")
    pos = np.empty(len(order), dtype=np.int64)
    pos[order] = np.arange(len(order))
    for (u, t) in edges:
        assert pos[u] < pos[t]
    # tiles partition [0, n) and stay inside one level group
    gl, lp = s.table("group_lvl"), s.table("level_ptr")
    tg = s.table("tile_group")
    assert tp[0] == 0 and tp[-1] == U.n and np.all(np.diff(tp) > 0)
    for t in range(len(tp) - 1):
        g = tg[t]
        assert lp[gl[g]] <= tp[t] and tp[t + 1] <= lp[gl[g + 1]]
    # same-class rows are write-disjoint (oracle pairwise check), class = (tile, colour)
    cls = (tile_of.astype(np.int64) * 4096 + sub).astype(np.int64)
    _, cls = np.unique(cls, return_inverse=True)
    assert oracle.write_conflicts(Up, cls.astype(np.int32)) == 0


@pytest.mark.parametrize("name,mk", GRAPHS)
@pytest.mark.parametrize("tile_work", [40, 300, 4096])
def test_schedule_conflict_free_bruteforce(name, mk, tile_work):
    U = mk()
    s = P.build_schedule(U, tile_work=tile_work, max_tile_window=256 if tile_work < 1000 else 6144)
    _check_schedule_bruteforce(U, s)


def test_schedule_small_windows_force_splits():
    U = gen.st27(7, 2, True)
    s = P.build_schedule(U, max_tile_window=128, tile_work=100000)
    st = s.stats
    assert st["max_tile_window"] <= 128
    _check_schedule_bruteforce(U, s)


def test_distance2_levels_groups_bruteforce():
    """Level groups of >= 2 levels coloured alternately are distance-2 independent
    across same-colour groups (corollary_dk)."""
    for U in (gen.lap2d(12), gen.random_symmetric(300, 3.0, 7), gen.knn(400, 6, 2)):
        s = P.build_schedule(U, tile_work=50)
        perm, inv = s.permutation()
        lp, gl = s.table("level_ptr"), s.table("group_lvl")
        grp_of_row = np.zeros(U.n, dtype=np.int64)
        for g in range(len(gl) - 1):
            grp_of_row[lp[gl[g]]:lp[gl[g + 1]]] = g
        assert np.all(np.diff(gl) >= 2) or len(gl) <= 3
        gp, ga = oracle.graph(U)
        # class = colour of the group, distinct per group: vertices in different
        # groups of the same colour must be distance-2 independent
        g_orig = grp_of_row[perm]
        viol = 0
        for colour in (0, 1):
            cls = np.where(g_orig % 2 == colour, g_orig, -1).astype(np.int32)
            # violations only count pairs in DIFFERENT groups of this colour
            same_group_pairs = oracle.distk_violations(gp, ga, 2, cls)
            cls2 = np.where(g_orig % 2 == colour, colour, -1).astype(np.int32)
            viol += oracle.distk_violations(gp, ga, 2, cls2) - same_group_pairs
        assert viol == 0


def test_determinism_and_islands():
    U = gen.spin(10, 4)
    s1, s2 = P.build_schedule(U), P.build_schedule(U)
    for t in ("dist", "tile_ptr", "tile_order", "row_subcolor", "dag_pred", "spill"):
        assert np.array_equal(s1.table(t), s2.table(t))
    assert s1.stats["n_components"] == 2
    lp = s1.table("level_ptr")
    assert 0 in np.diff(lp)  # empty separator level (island +2 rule)


def test_degenerate_inputs():
    U = gen.from_edges(1, [], [], [], [3.0])
    s = P.build_schedule(U)
    assert s.stats["n_tiles"] == 1
    U = gen.from_edges(5, [], [], [], np.arange(5.0))  # diagonal only: 5 islands
    s = P.build_schedule(U)
    assert s.stats["n_components"] == 5
    _check_schedule_bruteforce(U, s)
    # dense row (star) + missing diagonals
    n = 60
    U = gen.from_edges(n, [0] * (n - 1), list(range(1, n)), has_diag=(np.arange(n) % 3 != 0).astype(np.int8))
    s = P.build_schedule(U, tile_work=20)
    _check_schedule_bruteforce(U, s)


@pytest.mark.parametrize("name,mk", GRAPHS)
def test_rcm_levels_match_oracle(name, mk):
    """reorder = 2: the permutation is the oracle's reverse Cuthill-McKee order
    from the builder's roots; levels are the
    BFS levels of Eq. 5 counted from the far end, contiguous and ascending."""
    from oracle.race import rcm_order
    U = mk()
    s = P.build_schedule(U, reorder=2)
    roots = s.table("roots")
    gp, ga = oracle.graph(U)
    perm, inv = s.permutation()
    assert list(inv) == rcm_order(gp, ga, roots)
    d_or, tl = oracle.bfs_levels(gp, ga, roots)
    dist = s.table("dist")
    assert np.array_equal(dist, (tl - 1) - d_or)
    assert np.all(np.diff(dist[inv]) >= 0)
    assert np.array_equal(np.diff(s.table("level_ptr")), _levels_from_dist(dist))
    # the schedule is still conflict free and the permuted matrix is P A P^T
    rp, col, val = s.permuted_matrix()
    x = gen.vector_uniform(U.n, 3)
    yp = oracle.symmspmv(gen.UpperCSR(U.n, rp, col, val), x[inv])
    y = oracle.symmspmv(U, x)
    assert np.max(np.abs(yp - y[inv])) <= 1e-13 * max(1.0, np.max(np.abs(y)))
    with pytest.raises(Exception):
        P.build_schedule(U, reorder=2, cone_tiles=1)


@pytest.mark.parametrize("name,mk", GRAPHS)
def test_first_writer_flags(name, mk):
    """K8 (tiled_colored) stores for the first writer of a row (the writer tile
    of the lowest phase) and adds for the others: every row has exactly one
    first writer, among the tiles that write it (own tile or spill lists)."""
    U = mk()
    s = P.build_schedule(U)
    own_first = s.table("own_first").astype(np.int64)
    spill = s.table("spill").astype(np.int64) & 0xFFFFFFFF
    first = (spill >> 31) & 1
    tgt = spill & 0x7FFFFFFF
    cnt = own_first.copy()
    np.add.at(cnt, tgt[first == 1], 1)
    assert np.all(cnt == 1)
