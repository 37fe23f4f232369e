"""Per-tile pipeline timeline of CTA 0 of the tiled kernel (diagnostics).
Trace slots: 6 loader before empty-wait, 7 after, 0 block issued, 1 gather start
(stage free), 2 gather issued, 3 consumer has block + window, 4 passes+flush
done, 5 stage released."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen
import paper_1907_06487_b200 as P
from paper_1907_06487_b200 import _lib
cfg = sys.argv[1] if len(sys.argv) > 1 else "st27_128"
U, x = gen.make_config(cfg)
s = P.build_schedule(U)
plan = P.Plan(s, U, variant="tiled")
perm, inv = s.permutation()
xd = torch.from_numpy(x[inv].copy()).cuda(); yd = torch.empty_like(xd)
for _ in range(5): plan.run(xd, yd)
torch.cuda.synchronize()
L = C.CDLL(_lib.LIB_PATH)
L.symmspmv_debug_trace.argtypes = [C.c_void_p] * 5 + [C.c_int32]
cap = 4096
tr = np.zeros(cap * 8 + 16, dtype=np.uint64)
assert L.symmspmv_debug_trace(plan._h, C.c_void_p(xd.data_ptr()), C.c_void_p(yd.data_ptr()), None, tr.ctypes.data, cap) == 0
prof = tr[cap * 8: cap * 8 + 6].astype(np.float64)
tr = tr[:cap * 8].reshape(cap, 8).astype(np.int64)
n = int(np.count_nonzero(tr[:, 5])); tr = tr[:n]; t0 = tr[:, 6].min()
print("plan", plan.info(), "tiles of CTA0:", n, "span us", (tr[:, 5].max() - t0) / 1e3)
for nm, (a, b) in {"loader empty-wait": (6, 7), "loader issue": (7, 0), "gather issue (1->2)": (1, 2),
                   "stage free->consumer start (1->3)": (1, 3), "block issued->consumer start (0->3)": (0, 3),
                   "consumer passes+flush (3->4)": (3, 4)}.items():
    v = tr[:, b] - tr[:, a]
    print(f"{nm:38s} median {np.median(v):7.0f} ns  p90 {np.percentile(v, 90):7.0f}")
c3 = np.sort(tr[:, 3]); c4 = np.sort(tr[:, 4])
print("consumer start interval median (4 groups interleaved):", np.median(np.diff(c3)))
for i in range(8, 20):
    print(i, [int((v - t0) / 10) / 100 for v in tr[i, [6, 7, 0, 1, 2, 3, 4, 5]]])

if prof.sum() > 0:
    names = ["wait data", "row pass", "CSC pass", "flush", "release", "loop/other"]
    print("consumer warp-cycles (all CTAs):", {nm: f"{v / prof.sum() * 100:.1f}%" for nm, v in zip(names, prof)})
