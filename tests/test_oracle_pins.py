"""Pins of the CPU oracle against things other than itself (CPU only).

Each pin is chosen so that a plausible mistake in the oracle (a dropped
diagonal or transposed term, a wrong index, a transposed operand, a missing
island rule, a wrong level) fails at least one of them.
"""
import math

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.csgraph as csg

import gen
import oracle

U_EPS = 2.0 ** -53


def relinf(a, b):
    d = np.max(np.abs(np.asarray(a, dtype=np.float64) - np.asarray(b, dtype=np.float64))) if len(a) else 0.0
    s = np.max(np.abs(b)) if len(b) else 0.0
    return d / s if s > 0 else d


def scipy_full(U):
    """A = U + U^T - diag(U) with scipy (a library routine, independent of the oracle)."""
    Us = sp.csr_matrix((U.val, U.col, U.row_ptr), shape=(U.n, U.n))
    return (Us + Us.T - sp.diags(Us.diagonal())).tocsr()


SMALL = [
    lambda: gen.lap2d(7),
    lambda: gen.st27(5, 2, True),
    lambda: gen.spin(7, 4),
    lambda: gen.knn(150, 6, 3),
    lambda: gen.lap3d(5, 5, True),
    lambda: gen.random_symmetric(180, 6.0, 1),
    lambda: gen.random_symmetric(97, 2.5, 2, diag_frac=0.6),
    lambda: gen.banded_random(120, 9, 5.0, 3),
]


# --------------------------------------------------------------- SymmSpMV pins
@pytest.mark.parametrize("mk", SMALL)
def test_symmspmv_vs_dense_bruteforce(mk):
    """y = A x by the definition y_i = sum_j A_ij x_j on the dense matrix."""
    U = mk()
    x = gen.vector_uniform(U.n, 7)
    Ad = oracle.to_dense(U)
    y_dense = Ad @ x  # numpy, independent summation
    y = oracle.symmspmv(U, x)
    assert relinf(y, y_dense) <= 1e-14
    assert relinf(oracle.dense_matvec(Ad, x), y_dense) <= 1e-14


@pytest.mark.parametrize("mk", SMALL)
def test_symmspmv_vs_scipy_and_spmv_identity(mk):
    """SymmSpMV(U) == SpMV(A), A mirrored two independent ways."""
    U = mk()
    x = gen.vector_uniform(U.n, 11)
    A = scipy_full(U)
    y_sc = A @ x
    frp, fcol, fval = oracle.mirror(U)
    assert np.array_equal(frp, A.indptr.astype(np.int32))
    As = A.copy()
    As.sort_indices()
    assert np.array_equal(fcol, As.indices) and np.array_equal(fval, As.data)
    y_spmv = oracle.spmv(frp, fcol, fval, x)
    y = oracle.symmspmv(U, x)
    assert relinf(y, y_sc) <= 1e-13
    assert relinf(y_spmv, y_sc) <= 1e-13
    assert relinf(y, y_spmv) <= 1e-13


def test_laplacian_eigenpair_closed_form():
    """2-D 5-pt Laplacian, x_ij = sin(pi i/(N+1)) sin(pi j/(N+1)) -> A x = lambda x,
    lambda = 4 - 4 cos(pi/(N+1)) (north_star).  Backward-error bound (reading R6)."""
    N = 64
    U = gen.lap2d(N)
    x = gen.vector_sinsin(N)
    lam = 4.0 - 4.0 * math.cos(math.pi / (N + 1))
    assert abs(lam - 0.004671092670693433) < 1e-17
    y = oracle.symmspmv(U, x)
    err = np.max(np.abs(y - lam * x))
    assert err <= 8 * U_EPS * 8.0 * np.max(np.abs(x))
    # a dropped transposed term would leave O(1) errors:
    assert err < 1e-13


def test_spec_hand_cases():
    # [[2,1],[1,3]] . [1,1] = [3,4]
    U = gen.from_edges(2, [0], [1], [1.0], [2.0, 3.0])
    assert np.array_equal(oracle.symmspmv(U, np.array([1.0, 1.0])), [3.0, 4.0])
    # diagonal only -> b_i = d_i x_i
    d = np.array([1.5, -2.0, 3.25, 0.0])
    U = gen.from_edges(4, [], [], [], d)
    x = np.array([2.0, 3.0, -1.0, 9.0])
    assert np.array_equal(oracle.symmspmv(U, x), d * x)
    # single bond (0,1) = v with zero diagonal -> [v x1, v x0]
    U = gen.from_edges(2, [1], [0], [0.5], [0.0, 0.0])
    assert np.array_equal(oracle.symmspmv(U, np.array([3.0, 5.0])), [2.5, 1.5])
    # rows without a stored diagonal contribute no diagonal term (reading R1)
    U = gen.from_edges(3, [0, 1], [1, 2], [1.0, 2.0], [7.0, 7.0, 7.0], has_diag=[0, 1, 0])
    assert np.array_equal(oracle.symmspmv(U, np.array([1.0, 1.0, 1.0])), [1.0, 10.0, 2.0])


@pytest.mark.parametrize("mk", SMALL)
@pytest.mark.parametrize("nt", [1, 2, 3, 8])
def test_symmspmv_omp_thread_private(mk, nt):
    """OpenMP host baseline (thread-private target arrays):
    one thread is Alg. 2 bit for bit; any thread count is y = A x (dense brute force)."""
    U = mk()
    x = gen.vector_uniform(U.n, 11)
    y, used = oracle.symmspmv_omp(U, x, nt)
    assert used == min(nt, U.n)
    if nt == 1:
        assert np.array_equal(y, oracle.symmspmv(U, x))
    assert relinf(y, oracle.to_dense(U) @ x) <= 1e-14


def test_symmspmv_omp_edge_cases():
    U = gen.from_edges(1, [], [], [], [2.5])
    y, used = oracle.symmspmv_omp(U, np.array([4.0]), 4)
    assert used == 1 and y[0] == 10.0
    # a star: row 0 writes every row, so block 0's private array spans all of them
    U = gen.from_edges(50, [0] * 49, list(range(1, 50)))
    x = gen.vector_uniform(50, 2)
    y, _ = oracle.symmspmv_omp(U, x, 7)
    assert relinf(y, oracle.to_dense(U) @ x) <= 1e-14


def test_empty_and_single():
    U = gen.from_edges(0, [], [], [], np.zeros(0))
    assert oracle.symmspmv(U, np.zeros(0)).shape == (0,)
    U = gen.from_edges(1, [], [], [], [2.5])
    assert oracle.symmspmv(U, np.array([4.0]))[0] == 10.0


def test_linearity_and_long_double():
    U = gen.random_symmetric(300, 8.0, 5)
    x, z = gen.vector_uniform(U.n, 1), gen.vector_uniform(U.n, 2)
    a, b = 0.75, -1.25
    lhs = oracle.symmspmv(U, a * x + b * z)
    rhs = a * oracle.symmspmv(U, x) + b * oracle.symmspmv(U, z)
    assert relinf(lhs, rhs) <= 1e-13
    yl = oracle.symmspmv_ld(U, x)
    assert relinf(oracle.symmspmv(U, x), yl.astype(np.float64)) <= 1e-14


def test_write_conflicts_two_ways():
    for U in (gen.random_symmetric(60, 4.0, 9), gen.lap2d(6)):
        pairs = oracle.conflicting_row_pairs(U)
        cls = np.zeros(U.n, dtype=np.int32)
        assert oracle.write_conflicts(U, cls) == len(pairs)
        # each row its own class -> no conflicts
        assert oracle.write_conflicts(U, np.arange(U.n, dtype=np.int32)) == 0
    # hand case: rows 0 and 1 both write b[2]
    U = gen.from_edges(3, [0, 1], [2, 2])
    assert oracle.conflicting_row_pairs(U) == {(0, 2), (1, 2), (0, 1)}


# --------------------------------------------------------------- BFS level pins
def _levels(dist):
    tl = int(dist.max()) + 1 if len(dist) else 0
    return np.bincount(dist, minlength=tl)


def test_bfs_path_star_islands():
    # path 0-1-2-3-4, root 0 -> level_ptr = [0,1,2,3,4,5]
    gp, ga = oracle.graph(gen.path(5))
    dist, tl = oracle.bfs_levels(gp, ga, [0])
    assert tl == 5 and list(dist) == [0, 1, 2, 3, 4]
    # two islands {0-1}, {2-3}, root 0 -> L(2) empty
    gp, ga = oracle.graph(gen.from_edges(4, [0, 2], [1, 3]))
    dist, tl = oracle.bfs_levels(gp, ga, [0])
    assert list(dist) == [0, 1, 3, 4] and tl == 5
    # star with centre as root -> totalLvl = 2
    gp, ga = oracle.graph(gen.from_edges(6, [3] * 5, [0, 1, 2, 4, 5]))
    dist, tl = oracle.bfs_levels(gp, ga, [3])
    assert tl == 2 and dist[3] == 0 and sorted(dist) == [0, 1, 1, 1, 1, 1]


def test_bfs_grid_closed_forms():
    N = 9
    gp, ga = oracle.graph(gen.lap2d(N))
    dist, tl = oracle.bfs_levels(gp, ga, [0])
    assert tl == 2 * N - 1
    assert list(_levels(dist)) == [min(s + 1, 2 * N - 1 - s) for s in range(2 * N - 1)]
    # 7-pt N^3 from a corner: level s = #{(i,j,k) in [0,N)^3 : i+j+k = s}
    N = 7
    gp, ga = oracle.graph(gen.lap3d(N, 5, False))
    dist, tl = oracle.bfs_levels(gp, ga, [0])
    i, j, k = np.meshgrid(np.arange(N), np.arange(N), np.arange(N), indexing="ij")
    assert tl == 3 * N - 2
    assert np.array_equal(_levels(dist), np.bincount((i + j + k).ravel()))
    # 27-pt N^3 (unshuffled) from a corner: Chebyshev shells (d+1)^3 - d^3
    gp, ga = oracle.graph(gen.st27(N, 2, False))
    dist, tl = oracle.bfs_levels(gp, ga, [0])
    assert tl == N and list(_levels(dist)) == [(d + 1) ** 3 - d ** 3 for d in range(N)]


def test_bfs_spin_components_binomial():
    """i XOR (3<<b) keeps popcount parity: 2 components; levels C(L-1, d)."""
    L = 10
    U = gen.spin(L, 4)
    gp, ga = oracle.graph(U)
    ncomp, lab = csg.connected_components(scipy_full(U), directed=False)
    assert ncomp == 2
    dist, tl = oracle.bfs_levels(gp, ga, [0])
    comp0 = dist[lab == lab[0]]
    assert list(np.bincount(comp0)) == [math.comb(L - 1, d) for d in range(L)]
    # second island starts at level (L-1) + 2
    comp1 = dist[lab != lab[0]]
    assert comp1.min() == (L - 1) + 2
    assert tl == 2 * L + 1


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_bfs_vs_scipy_shortest_path_and_corollary(seed):
    U = gen.random_symmetric(200, 3.0, seed)
    gp, ga = oracle.graph(U)
    A = abs(scipy_full(U))
    root = 5
    D = csg.shortest_path(A, unweighted=True, directed=False)
    ncomp, lab = csg.connected_components(A, directed=False)
    dist, tl = oracle.bfs_levels(gp, ga, [root])
    comp = lab == lab[root]
    assert np.array_equal(dist[comp], D[root, comp].astype(np.int32))
    # |level(u) - level(v)| <= 1 on every edge inside a component
    rows = np.repeat(np.arange(U.n), np.diff(gp))
    assert np.all(np.abs(dist[rows] - dist[ga]) <= 1)
    # corollary_dk: level gap >= k+1 => distance > k
    for k in (1, 2, 3):
        gap = np.abs(dist[:, None] - dist[None, :]) >= k + 1
        assert np.all(D[gap] > k)


def test_distk_bruteforce_path():
    gp, ga = oracle.graph(gen.path(30))
    D = csg.shortest_path(abs(scipy_full(gen.path(30))), unweighted=True, directed=False)
    for k in (1, 2, 3):
        good = (np.arange(30) % (k + 1)).astype(np.int32)
        assert oracle.distk_violations(gp, ga, k, good) == 0
        bad = (np.arange(30) % k).astype(np.int32) if k > 1 else np.zeros(30, np.int32)
        expect = int(np.sum((D <= k) & (D > 0) & (bad[:, None] == bad[None, :])))
        got = oracle.distk_violations(gp, ga, k, bad)
        assert got == expect and got > 0


# ------------------------------------------------------------------ RCM pins
def test_rcm_textbook_cases():
    """Cuthill-McKee by hand: a path from an end is the
    natural order (RCM its reverse); a star from a leaf visits the centre,
    then the other leaves by index; children go by ascending degree."""
    from oracle.race import rcm_order
    gp, ga = oracle.graph(gen.path(6))
    assert rcm_order(gp, ga, [0]) == [5, 4, 3, 2, 1, 0]
    star = gen.from_edges(6, [0] * 5, [1, 2, 3, 4, 5])
    gp, ga = oracle.graph(star)
    assert rcm_order(gp, ga, [3]) == [5, 4, 2, 1, 0, 3]
    # root 0 with neighbours 1 (degree 3), 2 (degree 1), 3 (degree 2)
    U = gen.from_edges(6, [0, 0, 0, 1, 1, 3], [1, 2, 3, 4, 5, 4])
    gp, ga = oracle.graph(U)
    assert rcm_order(gp, ga, [0])[::-1][:4] == [0, 2, 3, 1]


@pytest.mark.parametrize("mk", [lambda: gen.lap2d(9), lambda: gen.knn(300, 6, 3), lambda: gen.st27(5, 2, True),
                                lambda: gen.random_symmetric(200, 6.0, 1)])
def test_rcm_vs_scipy(mk):
    """On a connected graph scipy's reverse_cuthill_mckee starts from a
    minimum-degree vertex (its choice among ties is its own) and orders
    children by degree, ties by index; the oracle from scipy's start vertex
    (the last vertex of its RCM order) must give the identical order."""
    from oracle.race import rcm_order
    U = mk()
    gp, ga = oracle.graph(U)
    A = sp.csr_matrix((np.ones(len(ga)), ga, gp), shape=(U.n, U.n))
    ncomp, _ = csg.connected_components(A, directed=False)
    assert ncomp == 1
    ref = csg.reverse_cuthill_mckee(A, symmetric_mode=True)
    root = int(ref[-1])
    assert np.diff(gp)[root] == np.diff(gp).min()
    assert rcm_order(gp, ga, [root]) == list(ref)


# ------------------------------------------------------- NEXT-4 sweep pins
def _spd_small():
    U = gen.random_symmetric(40, 5.0, 3)
    A = oracle.to_dense(U)
    # diagonally dominant SPD: GS and Kaczmarz converge, A^{-1} b is unique
    U = gen.from_edges(40, *np.nonzero(np.triu(A, 1)), A[np.triu_indices(40, 1)][np.triu(A, 1)[np.triu_indices(40, 1)] != 0],
                       np.abs(A).sum(1) + 1.0)
    return U


def test_gs_sweep_is_the_matrix_splitting():
    """One forward GS sweep in natural order is x' = (D + L)^{-1} (b - U_s x)
    (textbook splitting A = L + D + U_s; numpy triangular solve)."""
    import scipy.linalg as sl
    U = _spd_small()
    A = oracle.to_dense(U)
    rng = np.random.default_rng(1)
    b, x0 = rng.uniform(-1, 1, U.n), rng.uniform(-1, 1, U.n)
    x = oracle.sweep("gs", U, b, x0, np.arange(U.n, dtype=np.int32))
    ref = sl.solve_triangular(np.tril(A), b - np.triu(A, 1) @ x0, lower=True)
    assert relinf(x, ref) <= 1e-13


@pytest.mark.parametrize("kind", ["gs", "kacz"])
def test_sweeps_fix_the_solution_and_converge(kind):
    """A x* = b is a fixed point of both sweeps; symmetric sweeps converge to it."""
    U = _spd_small()
    A = oracle.to_dense(U)
    rng = np.random.default_rng(2)
    b = rng.uniform(-1, 1, U.n)
    xs = np.linalg.solve(A, b)
    order = rng.permutation(U.n).astype(np.int32)
    assert relinf(oracle.sweep(kind, U, b, xs, order, symmetric=True), xs) <= 1e-13
    x = np.zeros(U.n)
    res = []
    for _ in range(30):
        x = oracle.sweep(kind, U, b, x, order, symmetric=True)
        res.append(np.linalg.norm(A @ x - b))
    assert res[-1] < 1e-3 * res[0] and res[-1] <= np.linalg.norm(b) * 1e-4


def test_kacz_projects_onto_the_row():
    """eq:KACZ: after projecting onto row i, <A_i, x> = b_i,
    and x moved along A_i only."""
    U = _spd_small()
    A = oracle.to_dense(U)
    rng = np.random.default_rng(3)
    b, x0 = rng.uniform(-1, 1, U.n), rng.uniform(-1, 1, U.n)
    for i in (0, 7, 39):
        x = oracle.sweep("kacz", U, b, x0, np.array([i], dtype=np.int32))
        assert abs(A[i] @ x - b[i]) <= 1e-13 * (np.abs(A[i]) @ np.abs(x) + abs(b[i]))
        d = x - x0
        assert np.allclose(d, (d @ A[i]) / (A[i] @ A[i]) * A[i], atol=1e-14)


# --------------------------------------------------------------- matrix powers (NEXT-4)
@pytest.mark.parametrize("mk", SMALL[:6])
def test_matrix_powers_vs_dense_matrix_power(mk):
    """A^k x for k = 1..4 against numpy's matrix_power of the scipy-built dense
    A = U + U^T - diag(U) (library routines, independent of the oracle)."""
    U = mk()
    A = scipy_full(U).toarray()
    x = np.random.default_rng(7).uniform(-1, 1, U.n)
    Y = oracle.matrix_powers(U, x, 4)
    assert Y.shape == (4, U.n)
    for k in range(1, 5):
        ref = np.linalg.matrix_power(A, k) @ x
        scale = np.max(np.linalg.matrix_power(np.abs(A), k) @ np.abs(x))
        assert np.max(np.abs(Y[k - 1] - ref)) <= 1e-13 * scale, k


@pytest.mark.parametrize("p,q", [(3, 5), (30, 28)])
def test_matrix_powers_laplacian_modes(p, q):
    """2-D 5-pt Laplacian on N x N: x_ij = sin(p pi i/(N+1)) sin(q pi j/(N+1)) is an
    eigenvector, lambda = 4 - 2 cos(p pi/(N+1)) - 2 cos(q pi/(N+1)), so A^k x =
    lambda^k x (closed form; a low and a high mode).  Bound: x's own entries
    carry ~2u rounding (two sines and a product), amplified per step by
    ||A - lambda I||_inf <= 8 + |lambda|, plus each product's rounding:
    32 k u (8 + |lambda|)^k ||x||_inf."""
    N = 31
    U = gen.lap2d(N)
    i = np.arange(1, N + 1)
    x = np.outer(np.sin(p * np.pi * i / (N + 1)), np.sin(q * np.pi * i / (N + 1))).ravel()
    lam = 4 - 2 * math.cos(p * math.pi / (N + 1)) - 2 * math.cos(q * math.pi / (N + 1))
    Y = oracle.matrix_powers(U, x, 5)
    for k in range(1, 6):
        err = np.max(np.abs(Y[k - 1] - lam ** k * x))
        assert err <= 32 * k * U_EPS * (8.0 + abs(lam)) ** k * np.max(np.abs(x)), (k, err)
        # a dropped transposed term or a missing power leaves O(lambda^(k-1)) errors
        assert err < 1e-3 * abs(lam) ** (k - 1) * np.max(np.abs(x))


def test_matrix_powers_degenerate():
    U = gen.lap2d(6)
    x = np.random.default_rng(8).uniform(-1, 1, U.n)
    assert oracle.matrix_powers(U, x, 0).shape == (0, U.n)
    # diagonal-only matrix: A^k x = d^k x elementwise
    D = gen.from_edges(5, [], [], [], diag=[2.0, -1.0, 0.5, 3.0, 1.0])
    xd = np.array([1.0, 2.0, -1.0, 0.5, 4.0])
    d = np.array([2.0, -1.0, 0.5, 3.0, 1.0])
    Y = oracle.matrix_powers(D, xd, 3)
    for k in range(1, 4):
        assert np.array_equal(Y[k - 1], d ** k * xd)
