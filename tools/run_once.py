"""Run one variant once on a config with schedule overrides (diagnostics, e.g. under compute-sanitizer)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen, oracle
import paper_1907_06487_b200 as P
cfg, variant = sys.argv[1], sys.argv[2]
kw = {k: int(v) for k, v in (a.split("=") for a in sys.argv[3:])}
U, x = gen.make_config(cfg)
s = P.build_schedule(U, **kw)
perm, inv = s.permutation()
plan = P.Plan(s, U, variant=variant)
print("plan", plan.info(), flush=True)
xd = torch.from_numpy(x[inv].copy()).cuda(); yd = torch.empty_like(xd)
plan.run(xd, yd); torch.cuda.synchronize()
y = yd.cpu().numpy()[perm]
y_ref = oracle.symmspmv(U, x)
print("relinf", float(np.max(np.abs(y - y_ref)) / np.max(np.abs(y_ref))))
