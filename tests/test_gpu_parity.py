"""GPU parity: the CUDA path through the C ABI vs the CPU oracle (Alg. 2).

Bar (north_star): ||y_gpu - y_ref||_inf / ||y_ref||_inf <= 1e-12 in fp64;
the colored and tiled variants are bitwise deterministic run to run.
"""
import math
import os

import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu

TOL = 1e-12
VARIANTS = ("atomic", "colored", "tiled", "tiled_atomic", "colored_smem", "spmv", "tiled_colored")
# fp64 RED flushes: run-to-run summation order varies (reading R5)
NONDET = ("atomic", "tiled_atomic", "colored_smem")


def _torch():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: -m gpu tests need a B200")
    return torch


def relinf(a, b):
    s = np.max(np.abs(b)) if len(b) else 0.0
    d = np.max(np.abs(a - b)) if len(a) else 0.0
    return d / s if s > 0 else d


def run_gpu(U, x, variant, sched_kw=None, plan_kw=None, repeats=1):
    torch = _torch()
    import paper_1907_06487_b200 as P

    s = P.build_schedule(U, **(sched_kw or {}))
    plan = P.Plan(s, U, variant=variant, **(plan_kw or {}))
    perm, inv = s.permutation()
    xd = torch.from_numpy(x[inv].copy()).cuda()
    outs = []
    for _ in range(repeats):
        yd = torch.full((U.n,), float("nan"), dtype=torch.float64, device="cuda")
        plan.run(xd, yd)
        torch.cuda.synchronize()
        outs.append(yd.cpu().numpy()[perm])
    return outs, plan, s


SMALL = ["lap2d_64", "st27_24", "fem_knn_30k", "spin_14", "lap3d_40"]


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("name", SMALL)
def test_parity_small_configs(name, variant):
    U, x = gen.make_config(name)
    y_ref = oracle.symmspmv(U, x)
    outs, plan, _ = run_gpu(U, x, variant, repeats=3 if variant not in NONDET else 1)
    assert relinf(outs[0], y_ref) <= TOL
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])  # colored/tiled: bitwise deterministic
    assert plan.last_launches >= 1


@pytest.mark.parametrize("variant", VARIANTS)
def test_laplacian_eigenvector(variant):
    N = 64
    U = gen.lap2d(N)
    x = gen.vector_sinsin(N)
    lam = 4.0 - 4.0 * math.cos(math.pi / (N + 1))
    (y,), _, _ = run_gpu(U, x, variant)
    assert relinf(y, oracle.symmspmv(U, x)) <= TOL
    assert np.max(np.abs(y - lam * x)) <= 16 * 2.0 ** -53 * 8.0  # backward-error bound


EDGE = [
    ("single", lambda: gen.from_edges(1, [], [], [], [2.5])),
    ("diag_only", lambda: gen.from_edges(7, [], [], [], np.arange(1.0, 8.0))),
    ("no_diag_rows", lambda: gen.random_symmetric(700, 4.0, 11, diag_frac=0.5)),
    ("islands", lambda: gen.random_symmetric(900, 1.1, 12)),
    ("star", lambda: gen.from_edges(300, [0] * 299, list(range(1, 300)))),
    ("band_ragged", lambda: gen.banded_random(3001, 40, 9.0, 13)),
    ("path", lambda: gen.path(1000)),
]


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("name,mk", EDGE)
def test_parity_edge_cases(name, mk, variant):
    U = mk()
    x = gen.vector_uniform(U.n, 5)
    y_ref = oracle.symmspmv(U, x)
    outs, _, _ = run_gpu(U, x, variant, sched_kw=dict(tile_work=256))
    assert relinf(outs[0], y_ref) <= TOL


@pytest.mark.parametrize("variant", VARIANTS)
def test_many_tiles_small_windows(variant):
    """Tiny tiles => thousands of DAG edges / flush orderings on a small problem."""
    U, x = gen.make_config("st27_24")
    outs, _, s = run_gpu(U, x, variant, sched_kw=dict(tile_work=200, max_tile_window=512), repeats=3)
    assert s.stats["n_tiles"] > 300
    assert relinf(outs[0], oracle.symmspmv(U, x)) <= TOL
    if variant not in NONDET:
        assert all(np.array_equal(o, outs[0]) for o in outs)


def test_vector_order_original_and_host_path():
    torch = _torch()
    import paper_1907_06487_b200 as P

    U, x = gen.make_config("fem_knn_30k")
    y_ref = oracle.symmspmv(U, x)
    s = P.build_schedule(U)
    plan = P.Plan(s, U, variant="tiled", vec_order="original")
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    plan.run(xd, yd)
    torch.cuda.synchronize()
    assert relinf(yd.cpu().numpy(), y_ref) <= TOL
    yh = np.empty_like(x)
    plan.run_host(x, yh)
    assert relinf(yh, y_ref) <= TOL


def test_alias_and_mismatch_errors():
    torch = _torch()
    import paper_1907_06487_b200 as P

    U = gen.lap2d(16)
    s = P.build_schedule(U)
    plan = P.Plan(s, U, variant="tiled")
    xd = torch.zeros(U.n, dtype=torch.float64, device="cuda")
    with pytest.raises(P.SymmError) as e:
        plan.run(xd, xd)
    assert e.value.code == -9
    with pytest.raises(P.SymmError) as e:
        P.Plan(s, gen.lap2d(15))
    assert e.value.code == -8


FULL = ["st27_128", "fem_knn_4M", "spin_22", "lap3d_512"]


@pytest.mark.parametrize("name", FULL)
def test_parity_full_size(name):
    """Full BASELINE.json sizes, the bench launch configuration (tiled + atomic),
    compared against the full serial oracle (seconds even at 512^3)."""
    if name == "lap3d_512" and os.environ.get("SYMM_SKIP_512"):
        pytest.skip("SYMM_SKIP_512 set")
    torch = _torch()
    import paper_1907_06487_b200 as P

    U, x = gen.make_config(name)
    y_ref = oracle.symmspmv(U, x)
    s = P.build_schedule(U)
    perm, inv = s.permutation()
    plan = P.Plan(s, U, variant="auto", build_all=True)
    xd = torch.from_numpy(x[inv].copy()).cuda()
    yd = torch.empty_like(xd)
    for v in ("tiled", "tiled_atomic", "atomic", "colored", "colored_smem", "spmv", "tiled_colored"):
        yd.fill_(float("nan"))
        plan.run(xd, yd, variant=v)
        torch.cuda.synchronize()
        y = yd.cpu().numpy()[perm]
        assert relinf(y, y_ref) <= TOL, v
        if name == "st27_128" and v in ("tiled", "colored", "tiled_colored"):
            # deterministic variants: bitwise identical over 10 runs
            for _ in range(9):
                yd.fill_(float("nan"))
                plan.run(xd, yd, variant=v)
                torch.cuda.synchronize()
                assert np.array_equal(yd.cpu().numpy()[perm], y), v
    del plan


def test_tree_full_size_st27():
    """K7 (recursive tree, scheme 3) at the full config-2 size."""
    U, x = gen.make_config("st27_128")
    y_ref = oracle.symmspmv(U, x)
    outs, _, _ = run_gpu(U, x, "tree", sched_kw=dict(scheme=3, n_workers=296), repeats=2)
    assert relinf(outs[0], y_ref) <= TOL
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("variant", VARIANTS)
def test_empty_matrix(variant):
    """n = 0: plan and run succeed and launch nothing."""
    torch = _torch()
    import paper_1907_06487_b200 as P

    U = gen.from_edges(0, [], [], [], [])
    s = P.build_schedule(U)
    plan = P.Plan(s, U, variant=variant)
    xd = torch.zeros(0, dtype=torch.float64, device="cuda")
    yd = torch.zeros(0, dtype=torch.float64, device="cuda")
    plan.run(xd, yd)
    torch.cuda.synchronize()
    assert plan.last_launches == 0


def test_plans_share_kernel_attributes():
    """A plan built after another (smaller blocks, same ring depth) must not
    break runs of the first one (the kernels' shared-memory limit is a
    per-kernel attribute shared by every plan)."""
    torch = _torch()
    import paper_1907_06487_b200 as P

    Ua, xa = gen.make_config("st27_24")
    sa = P.build_schedule(Ua)
    pa = P.Plan(sa, Ua, variant="auto", build_all=True)
    Ub, xb = gen.make_config("lap2d_64")
    sb = P.build_schedule(Ub, tile_work=200, max_tile_window=256)
    pb = P.Plan(sb, Ub, variant="auto", build_all=True)
    for plan, s, U, x in ((pb, sb, Ub, xb), (pa, sa, Ua, xa), (pb, sb, Ub, xb)):
        perm, inv = s.permutation()
        xd = torch.from_numpy(x[inv].copy()).cuda()
        yd = torch.empty_like(xd)
        y_ref = oracle.symmspmv(U, x)
        for v in ("tiled", "tiled_atomic", "tiled_colored", "colored_smem"):
            yd.fill_(float("nan"))
            plan.run(xd, yd, variant=v)
            torch.cuda.synchronize()
            assert relinf(yd.cpu().numpy()[perm], y_ref) <= TOL, v


@pytest.mark.parametrize("ws", [2, 3])
@pytest.mark.parametrize("name", ["spin_14", "st27_24", "lap3d_40", "fem_knn_30k"])
def test_multirank_plans_emulated_on_one_gpu(name, ws):
    """Per-rank plans (own tiles only, shifted local vectors) run one after the
    other on one GPU; the halo exchange is emulated by copies.  Kernels never
    wait on each other (B200_PROFILING.md: no co-scheduled waiting ranks)."""
    torch = _torch()
    import paper_1907_06487_b200 as P
    from paper_1907_06487_b200.dist import halo_pieces

    U, x = gen.make_config(name)
    y_ref = oracle.symmspmv(U, x)
    s = P.build_schedule(U)
    perm, inv = s.permutation()
    xp = x[inv]
    b, h = s.partition(ws)
    yl = []
    nb_total = 0
    for r in range(ws):
        plan = P.Plan(s, U, variant="tiled_atomic", nranks=ws, rank=r)
        r0, he = plan.local_range()
        assert (r0, he) == (int(b[r]), int(h[r]))
        parts = plan.parts()
        nb_total += parts["boundary_tiles"]
        if r == ws - 1:
            assert parts["boundary_tiles"] == 0  # the last rank has no halo
        xd = torch.from_numpy(xp[r0:he].copy()).cuda()
        yd = torch.full_like(xd, float("nan"))
        # the overlapped sequence: interior part, (x halo arrives), boundary part
        plan.run_part("interior", xd, yd)
        plan.run_part("boundary", xd, yd)
        yl.append(yd)
    torch.cuda.synchronize()
    assert nb_total > 0
    # owner-side adds with the C-ABI halo-add kernel on device slices, in
    # ascending sender order (the exchange itself emulated by device copies)
    for q in range(ws):
        for p in range(q):
            for (qq, a, c) in halo_pieces(b, h, p):
                if qq == q:
                    buf = yl[p][a - int(b[p]):c - int(b[p])].clone()
                    P.halo_add(yl[q][a - int(b[q]):c - int(b[q])], buf)
    torch.cuda.synchronize()
    y = np.empty(U.n)
    for r in range(ws):
        r0, r1 = int(b[r]), int(b[r + 1])
        y[r0:r1] = yl[r][:r1 - r0].cpu().numpy()
    assert relinf(y[perm], y_ref) <= TOL


@pytest.mark.parametrize("scheme,block", [(1, 1), (2, 16), (2, 64)])
@pytest.mark.parametrize("variant", ["colored", "tiled_atomic", "tiled"])
def test_mc_abmc_schedules(scheme, block, variant):
    """NEXT-3: the MC / ABMC comparison schedules run through the same kernels."""
    U, x = gen.make_config("st27_24")
    y_ref = oracle.symmspmv(U, x)
    outs, _, _ = run_gpu(U, x, variant, sched_kw=dict(scheme=scheme, abmc_block=block))
    assert relinf(outs[0], y_ref) <= TOL


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["st27_24", "fem_knn_30k", "spin_14"])
@pytest.mark.parametrize("variant", VARIANTS)
def test_rcm_schedule(name, variant):
    """NEXT-2: RCM level construction (reorder = 2) runs through every kernel."""
    U, x = gen.make_config(name)
    y_ref = oracle.symmspmv(U, x)
    outs, _, _ = run_gpu(U, x, variant, sched_kw=dict(reorder=2))
    assert relinf(outs[0], y_ref) <= TOL


@pytest.mark.parametrize("name,nw", [("st27_24", 296), ("fem_knn_30k", 296), ("spin_14", 592), ("lap2d_64", 64),
                                     ("lap3d_40", 1184)])
def test_tree_variant(name, nw):
    """NEXT-2: the recursive RACE tree (scheme 3) in one persistent launch with
    tree-scoped counters (K7): matches the oracle, bitwise deterministic; the
    other variants run the same schedule."""
    U, x = gen.make_config(name)
    y_ref = oracle.symmspmv(U, x)
    outs, plan, s = run_gpu(U, x, "tree", sched_kw=dict(scheme=3, n_workers=nw), repeats=3)
    assert relinf(outs[0], y_ref) <= TOL
    assert all(np.array_equal(o, outs[0]) for o in outs[1:])
    for v in ("colored", "tiled_atomic", "tiled"):
        (y,), _, _ = run_gpu(U, x, v, sched_kw=dict(scheme=3, n_workers=nw))
        assert relinf(y, y_ref) <= TOL, v


def test_tree_variant_needs_tree_schedule():
    _torch()
    import paper_1907_06487_b200 as P

    U = gen.lap2d(16)
    with pytest.raises(P.SymmError):
        P.Plan(P.build_schedule(U), U, variant="tree")


@pytest.mark.parametrize("kind", ["gs", "kacz"])
@pytest.mark.parametrize("name,scheme", [("lap2d_64", 0), ("st27_24", 0), ("fem_knn_30k", 0), ("lap3d_40", 0),
                                         ("spin_14", 0), ("st27_24", 1), ("fem_knn_30k", 2), ("lap3d_40", 3)])
def test_sweep_matches_serial_oracle(name, scheme, kind):
    """NEXT-4: a symmetric GS / Kaczmarz sweep phase by phase on the GPU equals
    the serial oracle sweep in the plan's row order (rows of a phase commute),
    and the rows of every phase are distance-1 (GS) / distance-2 (KACZ)
    independent in the full graph (brute force)."""
    torch = _torch()
    import paper_1907_06487_b200 as P

    U, _ = gen.make_config(name)
    if kind == "gs" and name == "spin_14":
        pytest.skip("spin diagonals in (-2, 2): Gauss-Seidel divides by near-zero pivots")
    kw = dict(scheme=scheme)
    if scheme == 2:
        kw["abmc_block"] = 64
    if scheme == 3:
        kw["n_workers"] = 296
    s = P.build_schedule(U, **kw)
    perm, inv = s.permutation()
    sw = P.Sweep(s, kind)
    rows, ptr = sw.order()
    assert np.array_equal(np.sort(rows), np.arange(U.n))
    gp, ga = oracle.graph(U)
    for p in range(len(ptr) - 1):
        ph = inv[rows[ptr[p]:ptr[p + 1]]]  # original ids of the phase
        mark = np.zeros(U.n, dtype=np.int64)
        inph = np.zeros(U.n, dtype=bool)
        inph[ph] = True
        for v in ph:
            nb = ga[gp[v]:gp[v + 1]]
            if kind == "kacz":  # closed neighbourhoods of a phase are disjoint (distance >= 3)
                cl = np.concatenate([[v], nb])
                assert not mark[cl].any()
                mark[cl] = 1
            else:  # no two rows of a phase are adjacent (distance >= 2)
                assert not inph[nb].any()
    rng = np.random.default_rng(11)
    b, x0 = rng.uniform(-1, 1, U.n), rng.uniform(-1, 1, U.n)
    xd = torch.from_numpy(x0[inv].copy()).cuda()
    bd = torch.from_numpy(b[inv].copy()).cuda()
    sw.run(xd, bd, symmetric=True)
    torch.cuda.synchronize()
    x = xd.cpu().numpy()[perm]
    x_ref = oracle.sweep(kind, U, b, x0, inv[rows].astype(np.int32), symmetric=True)
    assert relinf(x, x_ref) <= TOL


def test_binding_rejects_bad_vectors():
    """The binding checks dtype, length, contiguity and device before any
    kernel touches the memory (a short y would be written past its end)."""
    torch = _torch()
    import paper_1907_06487_b200 as P

    U, x = gen.make_config("lap2d_64")
    s = P.build_schedule(U)
    plan = P.Plan(s, U, variant="tiled_atomic")
    xd = torch.zeros(U.n, dtype=torch.float64, device="cuda")
    with pytest.raises(P.SymmError):
        plan.run(xd, torch.zeros(U.n - 1, dtype=torch.float64, device="cuda"))
    with pytest.raises(TypeError):
        plan.run(xd, torch.zeros(U.n, dtype=torch.float32, device="cuda"))
    with pytest.raises(TypeError):
        plan.run(xd, torch.zeros(2 * U.n, dtype=torch.float64, device="cuda")[::2])
    with pytest.raises(P.SymmError):
        plan.run_host(x, np.zeros(U.n - 1))
    with pytest.raises(P.SymmError):
        plan.run_host(x.astype(np.float32), np.zeros(U.n))
    y = np.zeros(U.n)
    plan.run_host(x, y)
    assert relinf(y, oracle.symmspmv(U, x)) <= TOL


def _dist_worker(rank, ws, port, name, overlap, out):
    """One rank of DistSymmSpMV.run on cuda:0 with gloo (halo staged through
    host memory): the real exchange + run_part + halo-add-kernel path."""
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        import paper_1907_06487_b200 as P
        from paper_1907_06487_b200.dist import DistSymmSpMV

        torch.cuda.set_device(0)
        U, x = gen.make_config(name)
        s = P.build_schedule(U)
        perm, inv = s.permutation()
        D = DistSymmSpMV(s, U, overlap=overlap)
        xp = x[inv]
        xl = torch.full((D.n_local,), float("nan"), dtype=torch.float64, device="cuda")
        xl[:D.n_own] = torch.from_numpy(xp[D.row_begin:D.own_end].copy()).cuda()
        yl = torch.full_like(xl, float("nan"))
        D.run(xl, yl)
        torch.cuda.synchronize()
        assert np.array_equal(xl.cpu().numpy(), xp[D.row_begin:D.local_end])  # halo arrived
        y_ref = oracle.symmspmv(U, x)[inv]
        err = relinf(yl[:D.n_own].cpu().numpy(), y_ref[D.row_begin:D.own_end]) * \
            np.max(np.abs(y_ref[D.row_begin:D.own_end])) / np.max(np.abs(y_ref))
        out[rank] = (float(err), D.parts())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("overlap", [True, False])
@pytest.mark.parametrize("ws,name", [(2, "st27_24"), (3, "spin_14"), (2, "fem_knn_30k")])
def test_dist_symmspmv_run_gloo_one_gpu(ws, name, overlap):
    """DistSymmSpMV.run end to end (x-halo exchange, interior / boundary parts,
    y-halo exchange, halo-add kernel) with ws processes on one GPU.  The ranks'
    kernels never wait on each other; the exchange is host-side (gloo)."""
    _torch()
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_dist_worker, args=(ws, port, name, overlap, out), nprocs=ws, join=True)
    for r in range(ws):
        err, parts = out[r]
        assert err <= TOL, (r, err, parts)


# ------------------------------------------------------------------ matrix powers (NEXT-4)
def _powers_gpu(U, x, npow, variant, ld_pad=0, build_all=False):
    torch = _torch()
    import paper_1907_06487_b200 as P

    s = P.build_schedule(U)
    plan = P.Plan(s, U, variant=variant, build_all=build_all)
    perm, inv = s.permutation()
    xd = torch.from_numpy(x[inv].copy()).cuda()
    Y = torch.full((npow, U.n + ld_pad), float("nan"), dtype=torch.float64, device="cuda")
    plan.powers(xd, Y)
    torch.cuda.synchronize()
    return Y[:, :U.n].cpu().numpy()[:, perm], plan, xd, Y


@pytest.mark.parametrize("variant", ["tiled_atomic", "tiled", "tiled_colored", "colored", "atomic"])
@pytest.mark.parametrize("name", SMALL)
def test_matrix_powers_match_oracle(name, variant):
    """Y[k] = A^(k+1) x through symmspmv_powers vs oracle.matrix_powers, every
    power within 1e-12 (relative inf-norm), rows padded (ldy > n)."""
    U, x = gen.make_config(name)
    ref = oracle.matrix_powers(U, x, 4)
    Y, _, _, _ = _powers_gpu(U, x, 4, variant, ld_pad=5)
    for k in range(4):
        assert relinf(Y[k], ref[k]) <= TOL, (k, relinf(Y[k], ref[k]))


def test_matrix_powers_full_size_and_determinism():
    """Config 2 at full size, 3 powers with the bench variant; the deterministic
    K8 variant gives bitwise identical powers over repeats."""
    torch = _torch()
    U, x = gen.make_config("st27_128")
    ref = oracle.matrix_powers(U, x, 3)
    Y, plan, xd, Yd = _powers_gpu(U, x, 3, "auto", build_all=True)
    for k in range(3):
        assert relinf(Y[k], ref[k]) <= TOL, k
    plan.powers(xd, Yd, variant="tiled_colored")
    torch.cuda.synchronize()
    first = Yd.cpu().numpy()
    for _ in range(3):
        Yd.fill_(float("nan"))
        plan.powers(xd, Yd, variant="tiled_colored")
        torch.cuda.synchronize()
        assert np.array_equal(Yd.cpu().numpy(), first)


def test_matrix_powers_errors():
    torch = _torch()
    import paper_1907_06487_b200 as P

    U, x = gen.make_config("lap2d_64")
    s = P.build_schedule(U)
    plan = P.Plan(s, U)
    xd = torch.zeros(U.n, dtype=torch.float64, device="cuda")
    with pytest.raises(P.SymmError):
        plan.powers(xd, torch.zeros((2, U.n - 1), dtype=torch.float64, device="cuda"))  # ldy < n
    Y = torch.zeros((2, U.n), dtype=torch.float64, device="cuda")
    with pytest.raises(P.SymmError) as e:
        plan.powers(Y[1], Y)  # x inside Y
    assert e.value.code == -9
    plan.powers(xd, torch.zeros((0, U.n), dtype=torch.float64, device="cuda"))  # npow = 0: no-op
