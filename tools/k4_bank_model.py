"""Shared-memory wavefront model of K4's consumer loops (diagnostics).

Decodes the tile blocks (symm_tiled_format_dump) and counts, per warp lock step
and half warp, the wavefronts of every shared load the consumer issues:
8-B loads cost max bank-pair multiplicity per half warp, 4-B / 2-B loads the
max bank multiplicity (distinct 4-B words) per warp.  Usage:
  python tools/k4_bank_model.py CONFIG [ntiles_sample]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import gen  # noqa: E402
import paper_1907_06487_b200 as P  # noqa: E402
from test_tiled_format import dump  # noqa: E402


def wf8(addrs):  # byte addresses of active lanes of one half warp, 8-B loads
    if len(addrs) == 0:
        return 0
    pairs = {}
    for a in addrs:
        pairs.setdefault((a // 8) % 16, set()).add(a // 8)
    return max(len(v) for v in pairs.values())


def wf_small(addrs):  # 2-B / 4-B loads, whole warp: distinct 4-B words per bank
    if len(addrs) == 0:
        return 0
    banks = {}
    for a in addrs:
        banks.setdefault((a // 4) % 32, set()).add(a // 4)
    return max(len(v) for v in banks.values())


def model(desc, blocks, sample):
    b = blocks.tobytes()
    tot = {}
    ideal = {}
    rng = np.random.default_rng(0)
    for D in desc[rng.choice(len(desc), min(sample, len(desc)), replace=False)]:
        h = int(D["block_off"])
        T, S, nnz = int(D["nrows"]), int(D["nspill"]), int(D["nnz"])
        W = T + S
        if int(D["sorted"]):
            continue
        rseg = np.frombuffer(b, "<u4", T, h + 64).astype(int)
        start = np.zeros(T + 1, int)  # model uses (start, end) per row
        rend = (rseg & 0xFFFF) + (rseg >> 16)
        lcol = np.frombuffer(b, "<u2", nnz, h + int(D["o_lcol"])).astype(int)
        tptr = np.frombuffer(b, "<u2", W + 1, h + int(D["o_tptr"])).astype(int)
        tcsc = np.frombuffer(b, "<u4", int(tptr[W]), h + int(D["o_tidx"])).astype(int)
        ov, ol, ot = int(D["o_val"]), int(D["o_lcol"]), int(D["o_tidx"])
        xb = 1 << 20  # x window base (bank phase irrelevant, common shift)

        def add(k, v, i):
            tot[k] = tot.get(k, 0) + v
            ideal[k] = ideal.get(k, 0) + i

        for g0 in range(0, W, 32):
            lanes = range(g0, min(W, g0 + 32))
            rl = [(rseg[l] >> 16) if l < T else 0 for l in lanes]
            for j in range(max(rl)):
                act = [(l, (rseg[l] & 0xFFFF) + j) for l, n in zip(lanes, rl) if n > j]
                add("row_lcol", wf_small([ol + 2 * e for _, e in act]), 1)
                for half in (0, 1):
                    ah = [(l, e) for l, e in act if (l - g0) // 16 == half]
                    if not ah:
                        continue
                    add("row_val", wf8([ov + 8 * e for _, e in ah]), 1)
                    add("row_x", wf8([xb + 8 * lcol[e] for _, e in ah]), 1)
            cl = [tptr[l + 1] - tptr[l] for l in lanes]
            for j in range(max(cl)):
                act = [(l, tptr[l] + j) for l, n in zip(lanes, cl) if n > j]
                add("csc_rec", wf_small([ot + 4 * p for _, p in act]), 1)
                for half in (0, 1):
                    ah = [(l, p) for l, p in act if (l - g0) // 16 == half]
                    if not ah:
                        continue
                    add("csc_val", wf8([ov + 8 * (tcsc[p] & 0xFFFF) for _, p in ah]), 1)
                    add("csc_x", wf8([xb + 8 * (tcsc[p] >> 16) for _, p in ah]), 1)
    return tot, ideal


if __name__ == "__main__":
    U, x = gen.make_config(sys.argv[1])
    s = P.build_schedule(U)
    tot, ideal = model(*dump(s)[:2], int(sys.argv[2]) if len(sys.argv) > 2 else 400)
    T = sum(tot.values())
    I = sum(ideal.values())
    for k in tot:
        print(f"{k:9s} wavefronts {tot[k]:8d}  ideal {ideal[k]:8d}  excess {tot[k] - ideal[k]:8d}")
    print(f"total     wavefronts {T:8d}  ideal {I:8d}  excess {T - I:8d} ({(T - I) / T:.1%})")
