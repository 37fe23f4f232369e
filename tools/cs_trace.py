"""Event trace of CTA 0 of the colored_smem kernel (diagnostics)."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen
import paper_1907_06487_b200 as P
from paper_1907_06487_b200._lib import lib, check
name = sys.argv[1] if len(sys.argv) > 1 else "st27_128"
U, x = gen.make_config(name)
s = P.build_schedule(U); perm, inv = s.permutation()
plan = P.Plan(s, U, variant="colored_smem")
xd = torch.from_numpy(x[inv].copy()).cuda(); yd = torch.empty_like(xd)
for _ in range(5): plan.run(xd, yd)
torch.cuda.synchronize()
cap = 4096
buf = np.zeros(2 * cap + 1024 + 2048 + 64, dtype=np.uint64)
f = lib().symm_cs_debug_trace; f.argtypes = [C.c_void_p] * 5 + [C.c_int32]; f.restype = C.c_int
check(f(plan._h, C.c_void_p(xd.data_ptr()), C.c_void_p(yd.data_ptr()), None, buf.ctypes.data, cap))
ch = buf[:2 * cap].reshape(cap, 2).astype(np.int64); nch = int((ch[:, 1] > 0).sum())
tl = buf[2 * cap:2 * cap + 1024].reshape(256, 4).astype(np.int64); ntl = int((tl[:, 3] > 0).sum())
t0 = min(ch[0, 0], tl[0, 0])
print("chunks", nch, "tiles", ntl)
print("chunk issue times (us):", [round((ch[i, 1] - t0) / 1e3, 2) for i in range(min(nch, 40))])
print("chunk wait (us):", [round((ch[i, 1] - ch[i, 0]) / 1e3, 2) for i in range(min(nch, 40))])
print("issue interval mean (us):", round(float(np.diff(ch[:nch, 1]).mean()) / 1e3, 3), "total", round((ch[nch - 1, 1] - t0) / 1e3, 1))
for k in range(ntl):
    r = (tl[k] - t0) / 1e3
    print(f"tile {k}: start {r[0]:.2f} window {r[1]:.2f} colours {r[2]:.2f} flush {r[3]:.2f}  (colours {r[2]-r[1]:.2f} us)")

pc = buf[2 * cap + 1024:2 * cap + 1024 + 2048].reshape(512, 4).astype(np.int64)
cb = buf[2 * cap + 1024 + 2048:].astype(np.int64)
npc = int((pc[:, 1] > 0).sum())
print("tile 1 colour barriers (us):", [round((v - t0) / 1e3, 2) for v in cb if v > 0])
# chunk issue times for reference
for p in range(min(npc, 120)):
    w = pc[p, 3] & 0xff; chn = (pc[p, 3] >> 8) & 0xffffff; kk = pc[p, 3] >> 32
    print(f"piece {p}: colour {kk} warp {w} chunk {chn} (issued {(ch[chn,1]-t0)/1e3:.2f}) start {(pc[p,2]-t0)/1e3:.2f} landed {(pc[p,0]-t0)/1e3:.2f} released {(pc[p,1]-t0)/1e3:.2f}")
