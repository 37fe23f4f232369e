"""CPU checks of the K3/K4 tile-block format (no GPU).

The plan's tile blocks (paper_1907_06487_b200/csrc/capi.cpp, build_tiled_host)
are decoded here in numpy the way k_tiled walks them -- tile descriptor, lane
positions (work-sorted through sid[] or in slot order), each lane's row part
(rseg/lcol/val) then transposed part (tptr/tcsc), the x window of own rows and
spill targets, the flush targets -- and the decoded SymmSpMV is compared with
the oracle (Alg. 2).  Independently of the decode, every
stored off-diagonal entry must be read exactly once by its row's lane and once
by its column's lane, and the spill runs must place every target at a window id
of the right 16-B parity.  The GPU kernel itself is pinned by
tests/test_gpu_parity.py.
"""
import ctypes as C

import numpy as np
import pytest

import gen
import oracle

P = pytest.importorskip("paper_1907_06487_b200")
from paper_1907_06487_b200._lib import check, lib  # noqa: E402

DESC = np.dtype([("block_off", "<i8"), ("block_bytes", "<i4"), ("nrows", "<i4"), ("nspill", "<i4"), ("nnz", "<i4"),
                 ("row0", "<i4"), ("o_lcol", "<u2"), ("o_tidx", "<u2"), ("o_tptr", "<u2"), ("o_tgt", "<u2"),
                 ("o_sid", "<u2"), ("o_val", "<u2"), ("spill_off", "<i4"), ("run_off", "<i4"), ("nruns", "<i4"),
                 ("gather_runs", "<i4"), ("sorted", "<i4"), ("tgt_base", "<i4")])
assert DESC.itemsize == 64
RUN = np.dtype([("row", "<i4"), ("wid", "<i4"), ("len", "<i4"), ("pad", "<i4")])


def dump(s):
    f = lib().symm_tiled_format_dump
    f.argtypes = [C.c_void_p] + [C.c_void_p] * 5
    f.restype = C.c_int
    sizes = np.zeros(4, dtype=np.int64)
    check(f(s._h, sizes.ctypes.data, None, None, None, None))
    desc = np.zeros(int(sizes[0]), dtype=DESC)
    blocks = np.zeros(int(sizes[1]), dtype=np.uint8)
    runs = np.zeros(int(sizes[2]), dtype=RUN)
    targets = np.zeros(int(sizes[3]), dtype=np.int32)
    check(f(s._h, sizes.ctypes.data, desc.ctypes.data, blocks.ctypes.data, runs.ctypes.data, targets.ctypes.data))
    return desc, blocks, runs, targets


def decode_and_multiply(desc, blocks, runs, targets, n, xp):
    """y = A x from the tile blocks, walked like k_tiled (atomic flush); also
    returns the (row, col) pairs read by row parts and by transposed parts."""
    b = blocks.tobytes()
    y = np.zeros(n, dtype=np.float64)
    row_pairs, csc_pairs = [], []
    for D in desc:
        h = int(D["block_off"])
        hd = np.frombuffer(b, dtype=DESC, count=1, offset=h)[0]
        assert hd.tobytes() == D.tobytes()  # the descriptor travels with its block
        T, S, row0, nnz = int(D["nrows"]), int(D["nspill"]), int(D["row0"]), int(D["nnz"])
        W = T + S
        rseg = np.frombuffer(b, dtype="<u4", count=T, offset=h + 64).astype(np.int64)
        rst, rln = rseg & 0xFFFF, rseg >> 16  # own row segments: [rst, rst + rln)
        seg = np.zeros(nnz, dtype=np.int64)  # segments are disjoint (pads belong to none)
        for l in range(T):
            seg[rst[l]:rst[l] + rln[l]] += 1
        assert seg.max(initial=0) <= 1 and int(seg.sum()) == int(rln.sum())
        srt = int(D["sorted"])
        if not srt:
            lcol = np.frombuffer(b, dtype="<u2", count=nnz, offset=h + int(D["o_lcol"])).astype(np.int64)
            tptr = np.frombuffer(b, dtype="<u2", count=W + 1, offset=h + int(D["o_tptr"])).astype(np.int64)
            noff = int(tptr[W])
            tcsc = np.frombuffer(b, dtype="<u4", count=noff, offset=h + int(D["o_tidx"])).astype(np.int64)
        else:  # record lists: pseg[i] = start | len << 16 into rec (val index | x index << 16)
            pseg = np.frombuffer(b, dtype="<u4", count=W, offset=h + int(D["o_lcol"])).astype(np.int64)
            nrec = int(((pseg & 0xFFFF) + (pseg >> 16)).max(initial=0))
            rec = np.frombuffer(b, dtype="<u4", count=nrec, offset=h + int(D["o_tidx"])).astype(np.int64)
            lcol = np.full(nnz, -1, dtype=np.int64)
        if int(D["gather_runs"]) & 2:
            # single-run tile: no tgt[] in the block; window slot l >= T + npad flushes to row
            # tgt_base + l, the parity pad slot before it (if any) to nothing
            npad = (int(D["gather_runs"]) >> 2) & 1
            assert int(D["nruns"]) == 1 and int(D["o_tgt"]) + 15 >= int(D["o_val"]) - 16
            tgt = np.concatenate([np.full(npad, -1, dtype=np.int64), int(D["tgt_base"]) + T + np.arange(npad, S)])
        else:
            tgt = np.frombuffer(b, dtype="<i4", count=S, offset=h + int(D["o_tgt"])).astype(np.int64)
        assert np.array_equal(tgt, targets[int(D["spill_off"]):int(D["spill_off"]) + S])
        val = np.frombuffer(b, dtype="<f8", count=nnz, offset=h + int(D["o_val"]))
        if int(D["sorted"]):
            sid = np.frombuffer(b, dtype="<u2", count=W, offset=h + int(D["o_sid"])).astype(np.int64)
            assert np.array_equal(np.sort(sid), np.arange(W))  # a permutation of the window slots
        else:
            sid = np.arange(W)
        # the x window: own rows, then spill targets (pads read nothing)
        gid = np.concatenate([row0 + np.arange(T), tgt])
        xs = np.where(gid >= 0, xp[np.maximum(gid, 0)], 0.0)
        # spill runs: consecutive targets at consecutive window ids; gathered
        # runs start on a window id with the 16-B parity of their first row
        for R in runs[int(D["run_off"]):int(D["run_off"]) + int(D["nruns"])]:
            w, g, ln = int(R["wid"]), int(R["row"]), int(R["len"])
            assert T <= w and w + ln <= W
            assert np.array_equal(gid[w:w + ln], g + np.arange(ln))
            if int(D["gather_runs"]):
                assert (w - (g - row0)) % 2 == 0
        if not srt and nnz > int(rln.sum()):  # padded placement: the unrolled steps of a half warp's rows
            # (which begin after each lane's loop-length % 4 leftover steps) start on distinct bank pairs
            for g0 in range(0, W, 16):
                idx = [i for i in range(g0, min(W, g0 + 16)) if sid[i] < T]
                n_loop = [int(pseg[i] >> 16) if srt else int(rln[sid[i]]) for i in idx]
                # (unsorted loops unrolled by K4_UNROLL = 2 run a lane's len % 2 leftover step
                # first; the sorted record loop runs its blocks of 4 first, leftovers last)
                K4_UNROLL = 2
                res = [(int(D["o_val"]) // 8 + int(rst[sid[i]]) + (0 if srt else nl & (K4_UNROLL - 1))) % 16
                       for i, nl in zip(idx, n_loop)]
                assert len(set(res)) == len(res)
        if srt:
            # a lane's record list holds (val index | x window id) records in any order: row
            # records of own row l (entry (l, c), c >= l in upper storage, x window id of c) and
            # transposed records (entry (r, l), r < l an own row, x window id of r); the val array
            # of a sorted tile may be permuted (bank-pair colouring), rseg is not used
            uses = np.zeros(nnz, dtype=np.int64)
        for i in range(W):
            l = int(sid[i])
            acc = 0.0
            if srt:
                lst = rec[int(pseg[i] & 0xFFFF):int(pseg[i] & 0xFFFF) + int(pseg[i] >> 16)]
                for q in lst:
                    e, xi = int(q) & 0xFFFF, int(q) >> 16
                    uses[e] += 1
                    acc += val[e] * xs[xi]
                    if l < T and gid[xi] >= row0 + l:   # tmp += A[idx] x[col[idx]]
                        row_pairs.append((row0 + l, int(gid[xi])))
                    else:                               # b[col] += A[idx] x[row]
                        assert xi < T
                        csc_pairs.append((row0 + xi, int(gid[l])))
            else:
                if l < T:
                    for k in range(int(rst[l]), int(rst[l] + rln[l])):
                        acc += val[k] * xs[lcol[k]]              # tmp += A[idx] x[col[idx]]
                        row_pairs.append((row0 + l, int(gid[lcol[k]])))
                for q in tcsc[int(tptr[i]):int(tptr[i + 1])]:
                    q = int(q)
                    e, r = q & 0xFFFF, q >> 16
                    assert r < T and lcol[e] == l and rst[r] <= e < rst[r] + rln[r]
                    acc += val[e] * xs[r]                          # b[col] += A[idx] x[row]
                    csc_pairs.append((row0 + r, int(gid[l])))
            if gid[l] >= 0:
                y[gid[l]] += acc
            else:
                assert acc == 0.0
        if srt:
            assert uses.max(initial=0) <= 2  # an entry: once by its row's lane, once by its column's
    return y, row_pairs, csc_pairs


def permuted_pairs(s, U):
    rp = np.zeros(U.n + 1, dtype=np.int32)
    col = np.zeros(U.nnz, dtype=np.int32)
    val = np.zeros(U.nnz)
    check(lib().race_schedule_permuted_matrix(s._h, rp.ctypes.data, col.ctypes.data, val.ctypes.data))
    rows = np.repeat(np.arange(U.n), np.diff(rp))
    return sorted(zip(rows.tolist(), col.tolist())), sorted(zip(rows[col != rows].tolist(), col[col != rows].tolist()))


@pytest.mark.parametrize("name", ["lap2d_64", "lap3d_40", "st27_24", "spin_14", "fem_knn_30k"])
@pytest.mark.parametrize("gain", ["0.25", "0", "1"])
def test_tiled_format_decodes_to_oracle(name, gain, monkeypatch):
    monkeypatch.setenv("SYMM_SORT_GAIN", gain)  # sorted lanes: default rule / every tile / never
    U, x = gen.make_config(name)
    s = P.build_schedule(U)
    perm, inv = s.permutation()
    desc, blocks, runs, targets = dump(s)
    assert int(desc["nrows"].sum()) == U.n                      # tiles partition the rows
    assert np.array_equal(np.cumsum(desc["nrows"])[:-1], desc["row0"][1:])
    if gain == "1":
        assert not desc["sorted"].any()
    if gain == "0":  # every tile with > 32 slots whose record format fits the largest unsorted block
        assert desc["sorted"].any()
    y, row_pairs, csc_pairs = decode_and_multiply(desc, blocks, runs, targets, U.n, x[inv])
    y_ref = oracle.symmspmv(U, x)
    err = np.max(np.abs(y[perm] - y_ref)) / np.max(np.abs(y_ref))
    assert err <= 1e-13, err
    all_pairs, off_pairs = permuted_pairs(s, U)
    assert sorted(row_pairs) == all_pairs   # every stored entry once in its row's lane
    assert sorted(csc_pairs) == off_pairs   # every off-diagonal entry once in its column's lane


@pytest.mark.parametrize("name", ["fem_knn_30k", "st27_24"])
def test_tiled_format_val_colouring(name, monkeypatch):
    """Opt-in format of sorted tiles (SYMM_VAL_COLOR=1): records in free order, val permuted so
    that a half warp's lock-step val loads hit distinct bank pairs -- same product, every entry
    still read once by its row's lane and once by its column's lane."""
    monkeypatch.setenv("SYMM_VAL_COLOR", "1")
    monkeypatch.setenv("SYMM_SORT_GAIN", "0")
    U, x = gen.make_config(name)
    s = P.build_schedule(U)
    perm, inv = s.permutation()
    desc, blocks, runs, targets = dump(s)
    assert desc["sorted"].any()
    y, row_pairs, csc_pairs = decode_and_multiply(desc, blocks, runs, targets, U.n, x[inv])
    y_ref = oracle.symmspmv(U, x)
    assert np.max(np.abs(y[perm] - y_ref)) / np.max(np.abs(y_ref)) <= 1e-13
    all_pairs, off_pairs = permuted_pairs(s, U)
    assert sorted(row_pairs) == all_pairs
    assert sorted(csc_pairs) == off_pairs


def test_tiled_format_edge_cases():
    for U in (gen.from_edges(1, [], [], [], [2.5]), gen.path(200), gen.random_symmetric(300, 1.1, 12),
              gen.from_edges(120, [0] * 119, list(range(1, 120)))):
        x = np.random.default_rng(5).uniform(-1, 1, U.n)
        s = P.build_schedule(U)
        perm, inv = s.permutation()
        y, _, _ = decode_and_multiply(*dump(s), U.n, x[inv])
        y_ref = oracle.symmspmv(U, x)
        scale = max(np.max(np.abs(y_ref)), 1e-300)
        assert np.max(np.abs(y[perm] - y_ref)) / scale <= 1e-13
