"""Quick GPU parity check of one variant on the small configs (diagnostic tool)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen, oracle
import paper_1907_06487_b200 as P

v = sys.argv[1] if len(sys.argv) > 1 else "colored_smem"
for name in ["lap2d_64", "st27_24", "fem_knn_30k", "spin_14", "lap3d_40"]:
    U, x = gen.make_config(name)
    y_ref = oracle.symmspmv(U, x)
    s = P.build_schedule(U)
    perm, inv = s.permutation()
    plan = P.Plan(s, U, variant=v)
    xd = torch.from_numpy(x[inv].copy()).cuda()
    yd = torch.full_like(xd, float("nan"))
    plan.run(xd, yd)
    torch.cuda.synchronize()
    y = yd.cpu().numpy()[perm]
    err = float(np.max(np.abs(y - y_ref)) / np.max(np.abs(y_ref)))
    print(f"{v} {name}: n={U.n} relinf={err:.3e} {'OK' if err <= 1e-12 else 'FAIL'}", flush=True)
