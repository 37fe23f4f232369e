"""Per-phase clock64 profile of the colored_smem consumers (build with -DCS_PROF)."""
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
for _ in range(3): plan.run(xd, yd)
torch.cuda.synchronize()
cap = 16
buf = np.zeros(2 * cap + 1024 + 2048 + 64, dtype=np.uint64)
f = lib().symm_cs_debug_trace; f.argtypes = [C.c_void_p] * 5 + [C.c_int32]; f.restype = C.c_int
check(f(plan._h, C.c_void_p(xd.data_ptr()), C.c_void_p(yd.data_ptr()), None, buf.ctypes.data, cap))
v = buf[2 * cap + 1024 + 2048:2 * cap + 1024 + 2048 + 10].astype(np.float64)
names = ["slice setup", "piece wait", "piece body", "piece release", "slice end", "colour barrier", "tile start", "flush"]
tot = v[:8].sum()
print(f"pieces {v[8]:.0f} slices {v[9]:.0f}; total warp-cycles {tot:.3e}")
for i, nm in enumerate(names):
    print(f"{nm:15s} {v[i]/tot*100:5.1f}%  per piece {v[i]/max(v[8],1):8.1f} cyc  per slice {v[i]/max(v[9],1):8.1f}")
