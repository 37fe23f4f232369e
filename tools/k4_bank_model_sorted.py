"""Shared-memory wavefront model of K4's record loop over SORTED tiles (diagnostics).

Lane position i walks rec[jb .. jb+nt): q = rec[jb+u]; acc += val[q & 0xffff] * xs[q >> 16],
the 32 lanes of a warp in lock step.  Counts the wavefronts of the three loads per step
(8-B loads: max bank-pair multiplicity per half warp; 4-B loads: max distinct words per bank).
Usage: python tools/k4_bank_model_sorted.py CONFIG [ntiles_sample]"""
import os
import sys

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import gen  # noqa: E402
import paper_1907_06487_b200 as P  # noqa: E402
from k4_bank_model import wf8, wf_small  # noqa: E402
from test_tiled_format import dump  # noqa: E402


def model(desc, blocks, sample):
    b = blocks.tobytes()
    tot, ideal = {}, {}
    rng = np.random.default_rng(0)
    srt = desc[desc["sorted"] != 0]
    for D in srt[rng.choice(len(srt), min(sample, len(srt)), replace=False)]:
        h = int(D["block_off"])
        T, S = int(D["nrows"]), int(D["nspill"])
        W = T + S
        pseg = np.frombuffer(b, "<u4", W, h + int(D["o_lcol"])).astype(int)
        nrec = int(((pseg & 0xFFFF) + (pseg >> 16)).max(initial=0))
        rec = np.frombuffer(b, "<u4", nrec, h + int(D["o_tidx"])).astype(int)
        ov, ot = int(D["o_val"]), int(D["o_tidx"])
        xb = 1 << 20

        def add(k, v, i):
            tot[k] = tot.get(k, 0) + v
            ideal[k] = ideal.get(k, 0) + i

        for g0 in range(0, W, 32):
            lanes = list(range(g0, min(W, g0 + 32)))
            nt = [pseg[i] >> 16 for i in lanes]
            jb = [pseg[i] & 0xFFFF for i in lanes]
            for u in range(max(nt)):
                act = [(i - g0, jb[i - g0] + u) for i in lanes if nt[i - g0] > u]
                add("rec", wf_small([ot + 4 * p for _, p in act]), 1)
                for half in (0, 1):
                    ah = [p for ln, p in act if ln // 16 == half]
                    if not ah:
                        continue
                    add("val", wf8([ov + 8 * (rec[p] & 0xFFFF) for p in ah]), 1)
                    add("x", wf8([xb + 8 * (rec[p] >> 16) for p in ah]), 1)
    return tot, ideal


if __name__ == "__main__":
    U, x = gen.make_config(sys.argv[1])
    s = P.build_schedule(U)
    tot, ideal = model(*dump(s)[:2], int(sys.argv[2]) if len(sys.argv) > 2 else 200)
    T, I = sum(tot.values()), sum(ideal.values())
    for k in tot:
        print(f"{k:5s} wavefronts {tot[k]:8d}  ideal {ideal[k]:8d}  x{tot[k] / ideal[k]:.2f}")
    print(f"total wavefronts {T:8d}  ideal {I:8d}  excess {(T - I) / T:.1%}")
