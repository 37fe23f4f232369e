"""CPU checks of the K5 colored_smem format (no GPU).

The schedule builder's K5 blocks (paper_1907_06487_b200/csrc/cs_build.cpp) are
decoded here in numpy exactly the way k_cs walks them -- tile head, colour
ranges, slice records, JDS pieces, window ids -- and the decoded SymmSpMV is
compared with the oracle (Alg. 2).  Independently of the
decode, every colour of every tile is checked to be write-disjoint (the
distance-2 condition) and every stored entry of U is shown
to appear exactly once.  This pins the host-side format builder; the GPU
kernel itself is pinned by tests/test_gpu_parity.py.
"""
import ctypes as C

import numpy as np
import pytest

import gen
import oracle

P = pytest.importorskip("paper_1907_06487_b200")
from paper_1907_06487_b200._lib import check, lib  # noqa: E402

DESC = np.dtype([("head_off", "<i8"), ("head_bytes", "<i4"), ("row0", "<i4"), ("T", "<i4"), ("S", "<i4"),
                 ("ncolors", "<i4"), ("nslices", "<i4"), ("npieces", "<i4"), ("nchunks", "<i4"),
                 ("block_bytes", "<i4"), ("o_cslc", "<u2"), ("o_srec", "<u2"), ("o_ploc", "<u2"),
                 ("o_pw", "<u2"), ("o_tgt", "<u2"), ("o_clen", "<u2"), ("pad", "<u2", 4)])
assert DESC.itemsize == 64
RELEASE_UNITS = 4096


def dump(s, wcap=4096, chunk=24576, stages=4, V=1):
    f = lib().symm_cs_format_dump
    f.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32] + [C.c_void_p] * 5
    f.restype = C.c_int
    sizes = np.zeros(3, dtype=np.int64)
    check(f(s._h, wcap, chunk, stages, V, sizes.ctypes.data, None, None, None, None))
    desc = np.zeros(int(sizes[0]), dtype=DESC)
    coff = np.zeros(int(sizes[1]), dtype=np.int64)
    clen = np.zeros(int(sizes[1]), dtype=np.int32)
    blocks = np.zeros(int(sizes[2]), dtype=np.uint8)
    check(f(s._h, wcap, chunk, stages, V, sizes.ctypes.data, desc.ctypes.data, coff.ctypes.data, clen.ctypes.data,
            blocks.ctypes.data))
    return desc, coff, clen, blocks


def u16(b, off, n):
    return np.frombuffer(b, dtype="<u2", count=n, offset=off)


def decode_and_multiply(desc, coff, clen, blocks, n, xp, V=1):
    """y = A x from the K5 blocks, walked like k_cs; also returns the set of
    (row, col) pairs the blocks encode (global permuted ids) for coverage."""
    b = blocks.tobytes()
    y = np.zeros(n, dtype=np.float64)
    pairs = []
    chunk_index = 0
    for D in desc:
        h = int(D["head_off"])
        T, S, row0 = int(D["T"]), int(D["S"]), int(D["row0"])
        hdr_base = np.frombuffer(b, dtype="<i8", count=1, offset=h)[0]
        assert hdr_base == h + int(D["head_bytes"])  # chunks follow the head
        cslc = u16(b, h + int(D["o_cslc"]), int(D["ncolors"]) + 1)
        srec = np.frombuffer(b, dtype=np.uint32, count=4 * int(D["nslices"]), offset=h + int(D["o_srec"])).reshape(-1, 4)
        ploc = np.frombuffer(b, dtype="<u4", count=int(D["npieces"]), offset=h + int(D["o_ploc"]))
        pw = u16(b, h + int(D["o_pw"]), int(D["npieces"]))
        tgt = np.frombuffer(b, dtype="<i4", count=S, offset=h + int(D["o_tgt"]))
        nch = int(D["nchunks"])
        cl = np.frombuffer(b, dtype="<u4", count=nch, offset=h + int(D["o_clen"]))
        assert np.array_equal(cl, clen[chunk_index:chunk_index + nch])
        # release weights of the pieces of every chunk sum to RELEASE_UNITS
        for c in range(nch):
            assert int(pw[(ploc >> 20) == c].sum()) == RELEASE_UNITS
        gid = np.concatenate([row0 + np.arange(T), tgt]).astype(np.int64)  # window id -> global row
        xs = xp[gid]
        ys = np.zeros(T + S)

        def piece(loc):
            return int(coff[chunk_index + (int(loc) >> 20)]) + (int(loc) & 0xFFFFF)

        for kk in range(int(D["ncolors"])):
            written = set()
            for s in range(int(cslc[kk]), int(cslc[kk + 1])):
                ploc0, w1, w2, _ = (int(v) for v in srec[s])
                p0, nsteps, npc, m = w1 & 0xFFFF, w1 >> 16, w2 & 0xFF, (w2 >> 8) & 0xFF
                assert int(ploc[p0]) == ploc0 and 1 <= m <= 32 // V
                o = piece(ploc0)
                lane_rid = u16(b, o + 32, 32).astype(np.int64)
                lane_L = u16(b, o + 96, 32).astype(np.int64)
                lane_d = np.frombuffer(b, dtype="<f8", count=32, offset=o + 160)
                rid, L, d = lane_rid[::V][:m], lane_L[::V][:m], lane_d[::V][:m]
                assert np.all(np.diff(L) <= 0) and (int(L[0]) + V - 1) // V == nsteps  # lengths descend
                acc = d * xs[rid]
                for r in rid:  # a row's own slot is in its colour's write set
                    assert int(r) not in written
                    written.add(int(r))
                for kp in range(npc):
                    o = piece(ploc[p0 + kp])
                    eo = u16(b, o, 16).astype(np.int64)
                    nnzp = int(eo[15])
                    vo = o + (416 if kp == 0 else 32)
                    val = np.frombuffer(b, dtype="<f8", count=nnzp, offset=vo)
                    lc = u16(b, vo + 8 * nnzp, nnzp).astype(np.int64)
                    for u in range(16):
                        t = 16 * kp + u
                        start = 0 if u == 0 else int(eo[u - 1])
                        lanes = [ln for ln in range(32) if ln // V < m and L[ln // V] > t * V + ln % V]
                        assert int(eo[u]) - start == len(lanes)
                        for rank, ln in enumerate(lanes):  # JDS: rank among the step's valid lanes
                            i = ln // V
                            a, c = val[start + rank], int(lc[start + rank])
                            assert c not in written  # write-disjoint colour
                            written.add(c)
                            acc[i] += a * xs[c]           # tmp += A[idx] x[col]
                            ys[c] += a * xs[rid[i]]       # b[col] += A[idx] x[row]
                            pairs.append((row0 + int(rid[i]), int(gid[c])))
                ys[rid] += acc                            # b[row] += tmp
        np.add.at(y, gid, ys)
        chunk_index += nch
    return y, pairs


@pytest.mark.parametrize("name", ["lap2d_64", "st27_24", "spin_14", "fem_knn_30k"])
@pytest.mark.parametrize("wcap,V", [(512, 1), (4096, 1), (4096, 2), (2048, 4)])
def test_cs_format_decodes_to_oracle(name, wcap, V):
    U, x = gen.make_config(name)
    if U.n > 20000 and (wcap, V) != (4096, 1):
        pytest.skip("python decode time")
    s = P.build_schedule(U)
    perm, inv = s.permutation()
    desc, coff, clen, blocks = dump(s, wcap=wcap, V=V)
    assert int(desc["T"].sum()) == U.n                      # tiles partition the rows
    assert np.array_equal(np.cumsum(desc["T"])[:-1], desc["row0"][1:])
    xp = x[inv]
    y, pairs = decode_and_multiply(desc, coff, clen, blocks, U.n, xp, V)
    y_ref = oracle.symmspmv(U, x)
    err = np.max(np.abs(y[perm] - y_ref)) / np.max(np.abs(y_ref))
    assert err <= 1e-13, err
    # every stored off-diagonal entry of U' appears exactly once
    rp = np.zeros(U.n + 1, dtype=np.int32)
    col = np.zeros(U.nnz, dtype=np.int32)
    val = np.zeros(U.nnz)
    check(lib().race_schedule_permuted_matrix(s._h, rp.ctypes.data, col.ctypes.data, val.ctypes.data))
    rows = np.repeat(np.arange(U.n), np.diff(rp))
    off = col != rows
    want = sorted(zip(rows[off].tolist(), col[off].tolist()))
    assert sorted(pairs) == want


def test_cs_format_edge_cases():
    for U in (gen.from_edges(1, [], [], [], [2.5]), gen.path(200), gen.random_symmetric(300, 1.1, 12),
              gen.from_edges(120, [0] * 119, list(range(1, 120)))):
        x = np.random.default_rng(5).uniform(-1, 1, U.n)
        s = P.build_schedule(U)
        perm, inv = s.permutation()
        desc, coff, clen, blocks = dump(s)
        y, _ = decode_and_multiply(desc, coff, clen, blocks, U.n, x[inv])
        y_ref = oracle.symmspmv(U, x)
        scale = max(np.max(np.abs(y_ref)), 1e-300)
        assert np.max(np.abs(y[perm] - y_ref)) / scale <= 1e-13
