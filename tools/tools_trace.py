"""Diagnostics: per-tile pipeline timeline of CTA 0 of the tiled kernel."""
import ctypes as C
import sys

import numpy as np
import torch

import gen
import paper_1907_06487_b200 as P
from paper_1907_06487_b200 import _lib

cfg = sys.argv[1] if len(sys.argv) > 1 else "st27_128"
kw = {}
for a in sys.argv[2:]:
    k, v = a.split("=")
    kw[k] = int(v)
U, x = gen.make_config(cfg)
s = P.build_schedule(U, **kw)
plan = P.Plan(s, U, variant="tiled")
perm, inv = s.permutation()
xd = torch.from_numpy(x[inv].copy()).cuda()
yd = torch.empty_like(xd)
for _ in range(5):
    plan.run(xd, yd)
torch.cuda.synchronize()
L = C.CDLL(_lib.LIB_PATH)
L.symmspmv_debug_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32]
cap = 4096
tr = np.zeros(cap * 8, dtype=np.uint64)
rc = L.symmspmv_debug_trace(plan._h, C.c_void_p(xd.data_ptr()), C.c_void_p(yd.data_ptr()),
                            C.c_void_p(torch.cuda.current_stream().cuda_stream), tr.ctypes.data, cap)
assert rc == 0, rc
tr = tr.reshape(cap, 8).astype(np.int64)
n = int(np.count_nonzero(tr[:, 0]))
tr = tr[:n]
t0 = tr[:, 0].min()
print("plan", plan.info(), "tiles of CTA0:", n)
d = lambda a, b: tr[:, b] - tr[:, a]
names = ["issue->blk", "blk->gather_done", "gather_done->consumer", "passA", "passB+flush"]
for nm, (a, b) in zip(names, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5)]):
    v = d(a, b)
    print(f"{nm:24s} median {np.median(v):8.0f} ns  p90 {np.percentile(v, 90):8.0f}")
span = tr[:, 5].max() - t0
print("CTA0 span ns", span, "per tile", span / n)
print("issue interval median", np.median(np.diff(tr[:, 0])), "consumer end interval", np.median(np.diff(np.sort(tr[:, 5]))))
for i in list(range(0, 12)) + list(range(n // 2, n // 2 + 8)):
    print(i, [int(v - t0) for v in tr[i, :8]])
NS = plan.info()["tiled_stages"]
gap = tr[NS:, 0] - tr[:-NS, 5]
print("issue[k] - end[k-NS]: median", np.median(gap), "p10", np.percentile(gap, 10), "p90", np.percentile(gap, 90))
# consumer idle: time a group waits for its next tile's x
print("loader: before-wait -> after-wait median", np.median(tr[:, 7] - tr[:, 6]), " after-wait -> issued median", np.median(tr[:, 0] - tr[:, 7]), " issued -> next before-wait", np.median(tr[1:, 6] - tr[:-1, 0]))
for g in range(3):
    idx = np.arange(g, n, 3)
    idle = tr[idx[1:], 3] - tr[idx[:-1], 5]
    busy = tr[idx, 5] - tr[idx, 3]
    print(f"group {g}: busy median {np.median(busy):.0f} ns, idle-before-next median {np.median(idle):.0f} ns")
