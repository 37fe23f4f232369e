"""NEXT-2: the recursive RACE tree (race_config.scheme = 3), CPU checks.

The builder's tree (tree_* tables, final permutation) must equal the oracle's
step-by-step recursion (oracle.race.race_tree, §4.4.1-4.4.2)
started from the same stage-0 level groups; independently, every pair of
leaves that the tree lets run concurrently (same colour at their lowest common
ancestor) must be write-set disjoint (distance-2, brute
force), and eta must be §5's.
"""
import numpy as np
import pytest

import gen
import oracle
from oracle import race

P = pytest.importorskip("paper_1907_06487_b200")

CASES = [
    ("lap2d_64", lambda: gen.lap2d(64), 64),
    ("lap2d_64_w16", lambda: gen.lap2d(64), 16),
    ("st27_12", lambda: gen.st27(12, 2, True), 48),
    ("knn_3000", lambda: gen.knn(3000, 8, 3), 96),
    ("spin_12", lambda: gen.spin(12, 4), 64),
    ("islands", lambda: gen.random_symmetric(900, 1.3, 12), 32),
]


def tree_of(s):
    t = {k: s.table("tree_" + k) for k in ("parent", "cidx", "r0", "r1", "stage", "workers")}
    return [tuple(int(t[k][i]) for k in ("parent", "cidx", "r0", "r1", "stage", "workers")) for i in range(len(t["parent"]))]


@pytest.mark.parametrize("name,mk,nw", CASES)
def test_tree_matches_oracle_recursion(name, mk, nw):
    U = mk()
    s = P.build_schedule(U, scheme=3, n_workers=nw)
    nodes = tree_of(s)
    # stage 0 = the plain RACE schedule with the same worker count
    s0 = P.build_schedule(U, scheme=0, n_workers=nw)
    _, inv0 = s0.permutation()
    lp0, gl0, gw0 = s0.table("level_ptr"), s0.table("group_lvl"), s0.table("group_workers")
    groups = [(int(lp0[gl0[g]]), int(lp0[gl0[g + 1]]), int(gw0[g])) for g in range(len(gw0))]
    gp, ga = oracle.graph(U)
    nodes_or, inv_or = race.race_tree(gp, ga, inv0, groups, nw, 2, [0.8, 0.8, 0.5, 0.5])
    assert nodes == nodes_or
    _, inv = s.permutation()
    assert list(inv) == inv_or
    assert abs(s.stats["eta"] - race.tree_eta(nodes_or, nw)) <= 1e-12
    if name == "lap2d_64":
        assert max(n[4] for n in nodes) >= 1  # the recursion went below stage 0


@pytest.mark.parametrize("name,mk,nw", CASES)
def test_tree_concurrent_leaves_conflict_free(name, mk, nw):
    U = mk()
    s = P.build_schedule(U, scheme=3, n_workers=nw)
    nodes = tree_of(s)
    leaves = s.table("tree_leaf")
    lp = s.table("level_ptr")
    assert len(lp) == len(leaves) + 1 and lp[-1] == U.n
    # leaves partition the rows in position order; children partition parents
    assert all(nodes[v][2] == lp[i] and nodes[v][3] == lp[i + 1] for i, v in enumerate(leaves))
    kids = {}
    for i, nd in enumerate(nodes[1:], start=1):
        kids.setdefault(nd[0], []).append(i)
    for p, ch in kids.items():
        ch = sorted(ch, key=lambda c: nodes[c][1])
        assert [nodes[c][1] for c in ch] == list(range(len(ch)))
        assert nodes[ch[0]][2] == nodes[p][2] and nodes[ch[-1]][3] == nodes[p][3]
        assert all(nodes[a][3] == nodes[b][2] for a, b in zip(ch, ch[1:]))
    # ancestors path of every leaf: (node, child index taken below it)
    def path(v):
        out = []
        while nodes[v][0] >= 0:
            out.append((nodes[v][0], nodes[v][1]))
            v = nodes[v][0]
        return out[::-1]

    paths = [path(v) for v in leaves]

    def concurrent(a, b):
        pa, pb = paths[a], paths[b]
        i = 0
        while i < min(len(pa), len(pb)) and pa[i] == pb[i]:
            i += 1
        # lowest common ancestor pa[i][0] == pb[i][0]; branches pa[i][1], pb[i][1]
        return pa[i][1] % 2 == pb[i][1] % 2

    rp, col, _ = s.permuted_matrix()
    leaf_of = np.repeat(np.arange(len(leaves)), np.diff(lp))
    writers = {}
    for r in range(U.n):  # write set W(r) = {r} + upper columns
        for c in set([r] + list(col[rp[r]:rp[r + 1]])):
            writers.setdefault(int(c), set()).add(int(leaf_of[r]))
    for c, ls in writers.items():
        ls = sorted(ls)
        for i in range(len(ls)):
            for j in range(i + 1, len(ls)):
                assert not concurrent(ls[i], ls[j]), (c, ls[i], ls[j])


def test_tree_rejects_bad_config():
    U = gen.lap2d(8)
    with pytest.raises(Exception):
        P.build_schedule(U, scheme=3, cone_tiles=1)
    with pytest.raises(Exception):
        P.build_schedule(U, scheme=3, reorder=0)
