"""ORACLE — TEST INFRASTRUCTURE ONLY: RACE level aggregation, load balancing, eta.

Pure Python, step by step in the paper's order and notation.  Work per level
is an integer (rows, or nonzeros: "One can either balance the number of rows
... or the number of nonzeros").  All floating-point
decisions are taken in IEEE fp64 with the expression order written here; the
product's C++ builder must take the same decisions (readings R12-R14).
"""
from __future__ import annotations

import math


def _round_half_up(a: float) -> int:
    """[a], "the nearest integer to a"; ties round up (reading R12)."""
    return int(math.floor(a + 0.5))


def eps_aggregate(level_work, nthreads: int, k: int, eps: float):
    """§4.4.3 steps 1-3: form windows of successive levels.

    Step 1: w(L_s(i)) = nrows(L_s(i)) / nrows(T_{s-1}(j)) * nthreads(T_{s-1}(j)).
    Step 2: starting at the next untouched level, aggregate at least 2k levels
            until the combined weight a gives eps_ = 1 - |a - b| > eps, with
            b = max(1, [a]).  Then b is fixed and further levels are added
            while the combined weight stays <= b, i.e. while a' > a moves closer
            to b from below (reading R12: this is the reading under which both
            printed examples, 28/32 -> 7 levels and 54/32 -> 4 levels, hold).
    Step 3: continue with the next pair from the very next level.
    Leftover levels that cannot form a window of >= 2k levels, or whose
    window never meets the criterion, join/form the last window with
    b = max(1, [a]) (reading R12).

    Returns a list of (first_level, end_level, b) with end exclusive; each
    window is later split into one red and one blue level group.
    """
    L = len(level_work)
    total = 0
    for wl in level_work:
        total += int(wl)
    windows = []
    if L == 0:
        return windows
    if total == 0:
        return [(0, L, 1)]
    s = 0
    while s < L:
        if L - s < 2 * k:
            if windows:
                f, _, b = windows[-1]
                windows[-1] = (f, L, b)
            else:
                windows.append((s, L, 1))
            break
        cum = 0
        e = s
        accepted = False
        b = 1
        while e < L:
            cum += int(level_work[e])
            e += 1
            if e - s < 2 * k:
                continue
            a = float(cum) * float(nthreads) / float(total)
            b = max(1, _round_half_up(a))
            eps_ = 1.0 - abs(a - float(b))
            if eps_ > eps:
                accepted = True
                break
        if not accepted:
            a = float(cum) * float(nthreads) / float(total)
            b = max(1, _round_half_up(a))
            if windows and e - s < 2 * k:
                f, _, bb = windows[-1]
                windows[-1] = (f, L, bb)
            else:
                windows.append((s, L, b))
            break
        # b fixed: try a' > a closer to b (stay <= b)
        while e < L:
            nxt = cum + int(level_work[e])
            a2 = float(nxt) * float(nthreads) / float(total)
            if a2 <= float(b):
                cum = nxt
                e += 1
            else:
                break
        windows.append((s, e, b))
        s = e
    # a tail shorter than 2k levels joins the last window
    if len(windows) >= 2:
        f, e, b = windows[-1]
        if e - f < 2 * k:
            f0, _, b0 = windows[-2]
            windows[-2:] = [(f0, e, b0)]
    return windows


def split_window(level_work, first: int, end: int, k: int) -> int:
    """Initial red/blue split of one window (reading R13): the first level
    boundary m at which the red part holds at least half the window's work,
    clamped so both groups keep >= k levels ("keeping at least k levels",
    PAPER.md:1256-1258).  Windows with < 2k levels split at first + ceil/2."""
    nl = end - first
    if nl < 2 * k:
        return first + (nl + 1) // 2
    tot = 0
    for i in range(first, end):
        tot += int(level_work[i])
    cum = 0
    m = first
    while m < end:
        cum += int(level_work[m])
        m += 1
        if 2 * cum >= tot:
            break
    return min(max(m, first + k), end - k)


def _variance(T_ptr, worker, cum_work):
    """Lines 17-23 of Alg. 4 with reading R14:
    mean_c = sum_{g in c} size_g / sum_{g in c} worker_g, diff_g =
    size_g/worker_g - mean_c, var = dot(diff, diff)/len."""
    n_g = len(T_ptr) - 1
    size = [float(cum_work[T_ptr[g + 1]] - cum_work[T_ptr[g]]) for g in range(n_g)]
    tsw = [size[g] / float(worker[g]) for g in range(n_g)]
    sr = 0.0
    sb = 0.0
    wr = 0
    wb = 0
    for g in range(n_g):
        if g % 2 == 0:
            sr += size[g]
            wr += worker[g]
        else:
            sb += size[g]
            wb += worker[g]
    mean_r = sr / float(wr) if wr else 0.0
    mean_b = sb / float(wb) if wb else 0.0
    diff = [tsw[g] - (mean_r if g % 2 == 0 else mean_b) for g in range(n_g)]
    var = 0.0
    for g in range(n_g):
        var += diff[g] * diff[g]
    var /= float(n_g)
    return var, diff


def _shift(T_ptr, donor: int, receiver: int):
    """shift(T_ptr, d, r) (reading R13): move one level across
    every boundary between donor d and receiver r, so the donor loses one
    level, the receiver gains one, intermediate groups keep their count."""
    if donor < receiver:
        for j in range(donor + 1, receiver + 1):
            T_ptr[j] -= 1
    elif donor > receiver:
        for j in range(receiver + 1, donor + 1):
            T_ptr[j] += 1


def _argsort_stable(vals):
    return sorted(range(len(vals)), key=lambda i: (vals[i], i))


def alg4_balance(T_ptr, worker, level_work, kmin: int = 2, max_iter: int = 1_000_000, trace=None):
    """Alg. 4 "Load Balancing for two sweep, distance-2, two colors"
    (PAPER.md:2422-2494), literal loop structure; `> 2` is read as `> kmin`
    (at least k levels must remain).  Group g's color is
    g % 2.  Returns (T_ptr, var_history); if `trace` is a list, T_ptr at the
    top of every outer iteration (line 17, before update) is appended to it."""
    T_ptr = list(T_ptr)
    n_g = len(T_ptr) - 1
    cum = [0]
    for wl in level_work:
        cum.append(cum[-1] + int(wl))
    hist = []
    exit_ = False
    it = 0
    while not exit_ and it < max_iter:
        it += 1
        if trace is not None:
            trace.append(list(T_ptr))
        var, diff = _variance(T_ptr, worker, cum)
        hist.append(var)
        absRankIdx = _argsort_stable([-abs(d) for d in diff])
        rankIdx = _argsort_stable(diff)
        currRank = 0
        newVar = var
        old = list(T_ptr)
        while newVar >= var:
            T_ptr = list(old)
            fail = True
            g = absRankIdx[currRank]
            if diff[g] < 0:
                acquire = -1
                for el in reversed(rankIdx):
                    if el != g and (T_ptr[el + 1] - T_ptr[el]) > kmin:
                        acquire = el
                        fail = False
                        break
                if not fail:
                    _shift(T_ptr, acquire, g)
            elif (T_ptr[g + 1] - T_ptr[g]) > kmin:
                give = rankIdx[0]
                if give != g:
                    fail = False
                    _shift(T_ptr, g, give)
            if not fail:
                newVar, _ = _variance(T_ptr, worker, cum)
            if currRank == n_g - 1 and newVar >= var:
                T_ptr = list(old)
                exit_ = True
                break
            currRank += 1
    return T_ptr, hist


def nrows_eff(node):
    """§5 effective row count.  A node is an int (leaf
    workload) or a list of children alternating colors: nrowsEff = max over
    even-indexed children + max over odd-indexed children."""
    if isinstance(node, (int, float)):
        return node
    even = [nrows_eff(c) for c in node[0::2]]
    odd = [nrows_eff(c) for c in node[1::2]]
    return (max(even) if even else 0) + (max(odd) if odd else 0)


def eta(nrows_total, root, nthreads: int) -> float:
    """η = nrows_total / (nrowsEff(T_{-1}(0)) × nthreads)."""
    return float(nrows_total) / (float(nrows_eff(root)) * float(nthreads))


def rcm_order(g_ptr, g_adj, roots):
    """Reverse Cuthill-McKee order (PAPER.md:1052-1053 names RCM as RACE's
    alternative level construction; PAPER.md:2026, 2047, 2199 use it).
    Cuthill-McKee: a BFS from each root in turn (one per connected component,
    in the given order) that appends the unvisited neighbours of the vertex
    being expanded by ascending degree, ties by ascending index; the reverse
    of the whole visit order is RCM.  Returns the RCM order (position ->
    vertex) as a list.  Pure Python, for test-sized graphs."""
    n = len(g_ptr) - 1
    deg = [int(g_ptr[v + 1]) - int(g_ptr[v]) for v in range(n)]
    seen = [False] * n
    order = []
    for r in roots:
        r = int(r)
        if seen[r]:
            continue
        seen[r] = True
        queue = [r]
        head = 0
        while head < len(queue):
            u = queue[head]
            head += 1
            new = [int(v) for v in g_adj[int(g_ptr[u]):int(g_ptr[u + 1])] if not seen[int(v)]]
            new = sorted(set(new), key=lambda v: (deg[v], v))
            for v in new:
                seen[v] = True
                queue.append(v)
        order.extend(queue)
    return order[::-1]


def race_tree(g_ptr, g_adj, inv, groups, nthreads: int, k: int, eps_list):
    """The recursive RACE tree (§4.4.1-4.4.2), step by step.

    inv: position -> vertex after the stage-0 level permutation; groups: the
    stage-0 level groups T_0(j) as (first position, end position, workers).
    A level group T_s(j) with more than one worker is refined: (1) levels are
    constructed on the subgraph of T_s(j) plus its distance-1 neighbourhood
    (distance-(k-1) for k = 2), one BFS per island in the
    group's current order (root = its first unvisited group vertex, reading
    R29), a new island starting two levels further;
    (2) only the vertices of T_s(j) are kept in the new levels L_{s+1}
     and the group is re-permuted in that order
    (PAPER.md:1489-1491); (3) eps_{s+1} aggregation of
    the new levels with the group's workers (rows as the workload, reading
    R30), the red/blue split and Alg. 4 give T_{s+1}(:).  A group that yields
    fewer than two non-empty level groups stays a leaf (reading R31).
    Returns (nodes, inv): nodes[i] = (parent, child index, first, end, stage,
    workers), node 0 = T_{-1}(0), children listed after their parent."""
    inv = [int(v) for v in inv]
    n = len(inv)
    nodes = [(-1, 0, 0, n, -1, int(nthreads))]
    for j, (a, b, w) in enumerate(groups):
        nodes.append((0, j, int(a), int(b), 0, int(w)))
    i = 1
    while i < len(nodes):
        _, _, p0, p1, st0, w = nodes[i]
        node_id, i = i, i + 1
        st = st0 + 1
        if w <= 1 or p1 - p0 < 2:
            continue
        G = set(inv[p0:p1])
        H = set(G)
        for v in inv[p0:p1]:
            H.update(int(u) for u in g_adj[int(g_ptr[v]):int(g_ptr[v + 1])])
        level = {}
        bfs = []
        maxL = -1
        for root in inv[p0:p1]:               # (1) one BFS per island
            if root in level:
                continue
            level[root] = 0 if maxL < 0 else maxL + 2
            queue = [root]
            h = 0
            while h < len(queue):
                u = queue[h]
                h += 1
                maxL = max(maxL, level[u])
                for v in g_adj[int(g_ptr[u]):int(g_ptr[u + 1])]:
                    v = int(v)
                    if v in H and v not in level:
                        level[v] = level[u] + 1
                        queue.append(v)
            bfs.extend(queue)
        keep = [v for v in bfs if v in G]    # (2) the group's own vertices
        lw = [0] * (maxL + 1)
        for v in keep:
            lw[level[v]] += 1
        eps = eps_list[min(st, len(eps_list) - 1)]
        wins = eps_aggregate(lw, w, k, eps)  # (3)
        T, wk = [], []
        if wins:
            T.append(wins[0][0])
        for (f, e, b) in wins:
            T += [split_window(lw, f, e, k), e]
            wk += [b, b]
        if len(T) >= 3:
            T, _ = alg4_balance(T, wk, lw, kmin=k)
        inv[p0:p1] = keep
        sizes = [sum(lw[T[j]:T[j + 1]]) for j in range(len(T) - 1)]
        if sum(1 for c in sizes if c > 0) < 2:
            continue
        a = p0
        for j, c in enumerate(sizes):
            nodes.append((node_id, j, a, a + c, st, wk[j]))
            a += c
    return nodes, inv


def tree_eta(nodes, nthreads: int) -> float:
    """§5 eta of a tree given as race_tree's node list (rows as the workload):
    nested lists of children for nrows_eff."""
    kids = {i: [] for i in range(len(nodes))}
    for i, nd in enumerate(nodes[1:], start=1):
        kids[nd[0]].append(i)

    def build(i):
        if not kids[i]:
            return nodes[i][3] - nodes[i][2]
        ch = sorted(kids[i], key=lambda c: nodes[c][1])
        return [build(c) for c in ch]

    return eta(nodes[0][3] - nodes[0][2], build(0), nthreads)
