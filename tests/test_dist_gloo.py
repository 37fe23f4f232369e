"""Multi-rank path on CPU (gloo, world_size 2 and 3): the row-block partition
(`race_schedule_partition`) and the halo exchange (`dist.HaloExchange`) of the
product, with the per-rank multiply done by the oracle on the rank's rows.
The union of all ranks' own rows must equal the full oracle result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import oracle
import paper_1907_06487_b200 as P
from paper_1907_06487_b200.dist import HaloExchange, halo_pieces


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_rows_matrix(rp, col, val, r0, r1, n_loc):
    """Rows [r0, r1) of the permuted upper CRS, columns shifted by -r0, as an
    (n_loc x n_loc) upper matrix: its Alg. 2 product gives exactly the
    contributions of these rows to y[r0 : r0 + n_loc)."""
    e0, e1 = rp[r0], rp[r1]
    rp_l = np.zeros(n_loc + 1, dtype=np.int32)
    rp_l[1:r1 - r0 + 1] = rp[r0 + 1:r1 + 1] - e0
    rp_l[r1 - r0 + 1:] = e1 - e0
    return gen.UpperCSR(n_loc, rp_l, (col[e0:e1] - r0).astype(np.int32), val[e0:e1].copy())


def _host_add(dst, buf):
    """Owner-side halo add for the CPU test (on GPUs: the C-ABI halo-add kernel)."""
    dst.add_(buf)


def _worker(rank, ws, port, name, kw, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        U, x = gen.make_config(name) if isinstance(name, str) else name()
        s = P.build_schedule(U, **kw)
        perm, inv = s.permutation()
        rp, col, val = s.permuted_matrix()
        bounds, halo = s.partition(ws)
        r0, r1, he = int(bounds[rank]), int(bounds[rank + 1]), int(halo[rank])
        xp = x[inv]
        # the rank holds only its own slice of x; the halo must arrive by exchange
        x_loc = torch.full((he - r0,), float("nan"), dtype=torch.float64)
        x_loc[:r1 - r0] = torch.from_numpy(xp[r0:r1])
        hx = HaloExchange(bounds, halo, rank)
        hx.exchange_x(x_loc)
        assert not torch.isnan(x_loc).any()
        assert np.array_equal(x_loc.numpy(), xp[r0:he])
        Ul = _rank_rows_matrix(rp, col, val, r0, r1, he - r0)
        y_loc = torch.from_numpy(oracle.symmspmv(Ul, x_loc.numpy()))
        hx.reduce_y(y_loc, add=_host_add)
        y_full = oracle.symmspmv(U, x)[inv]
        err = float(np.max(np.abs(y_loc.numpy()[:r1 - r0] - y_full[r0:r1]))) / float(np.max(np.abs(y_full)))
        out[rank] = (err, r0, r1, he, hx.halo_bytes())
    finally:
        dist.destroy_process_group()


CASES = [
    ("lap3d_40", {}),
    ("spin_14", {}),                       # disconnected, wide levels: halo may span ranks
    ("st27_24", {"tile_work": 200}),
    ("fem_knn_30k", {}),
]


@pytest.mark.parametrize("ws", [2, 3])
@pytest.mark.parametrize("name,kw", CASES)
def test_gloo_row_block_halo(ws, name, kw):
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(ws, port, name, kw, out), nprocs=ws, join=True)
    res = [out[r] for r in range(ws)]
    assert res[0][1] == 0
    for r in range(ws - 1):
        assert res[r][2] == res[r + 1][1]  # contiguous blocks
    for err, r0, r1, he, hb in res:
        assert err <= 1e-13, (err, r0, r1)
        assert he >= r1


def test_partition_properties():
    U, _ = gen.make_config("spin_14")
    s = P.build_schedule(U)
    tp = s.table("tile_ptr")
    rp, col, _ = s.permuted_matrix()
    for ws in (1, 2, 3, 8):
        b, h = s.partition(ws)
        assert b[0] == 0 and b[-1] == U.n and np.all(np.diff(b) >= 0)
        assert set(b.tolist()) <= set(tp.tolist())  # whole tiles per rank
        for r in range(ws):
            e0, e1 = rp[b[r]], rp[b[r + 1]]
            mx = int(col[e0:e1].max()) + 1 if e1 > e0 else b[r + 1]
            assert h[r] >= max(mx, b[r + 1])  # every column a rank touches is inside its local range
        if ws > 1:
            nz = [rp[b[r + 1]] - rp[b[r]] for r in range(ws)]
            assert max(nz) <= 1.5 * U.nnz / ws + rp[-1] / len(tp) * 2  # balanced up to a tile
    # halo spanning more than one rank is representable
    assert halo_pieces([0, 10, 20, 30], [25, 30, 30], 0) == [(1, 10, 20), (2, 20, 25)]
