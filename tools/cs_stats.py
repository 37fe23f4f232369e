"""Host-side statistics of the K5 colored_smem format (no GPU)."""
import ctypes as C, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen
import paper_1907_06487_b200 as P
from paper_1907_06487_b200._lib import lib, check

name = sys.argv[1]
U, x = gen.make_config(name)
t0 = time.time(); s = P.build_schedule(U); tb = time.time() - t0
L = lib(); f = L.symm_cs_format_stats; f.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]; f.restype = C.c_int
for w in [int(a) for a in sys.argv[2].split(",")]:
    for ch in [int(a) for a in (sys.argv[3] if len(sys.argv) > 3 else "24576").split(",")]:
        out = np.zeros(13, dtype=np.int64)
        t0 = time.time()
        NS = int(os.environ.get('NS', '4'))
        check(f(s._h, w, ch, NS, int(os.environ.get('V', '1')), out.ctypes.data))
        nt, Wc, sc, sl, steps, nnz, sp, by, mcc, rows, conf, heads, hcap = out.tolist()
        print(f"{name} W={w} chunk={ch}: tiles={nt} Wcap={Wc} Hcap={hcap} colours/tile={sc/nt:.1f} rows/colour={rows/sc:.1f} "
              f"slices/colour={sl/sc:.2f} lane-util={nnz/max(16*steps,1):.3f} bank-conflict-steps={conf/max(steps,1):.4f} "
              f"spill/row={sp/rows:.3f} B/nnz_u={by/U.nnz:.2f} head B/row={heads/rows:.2f} colour-span={mcc} "
              f"build={time.time()-t0:.1f}s", flush=True)
