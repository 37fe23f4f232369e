"""Run one variant N times on a config (diagnostics under ncu: launch lists, DRAM bytes)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen
import paper_1907_06487_b200 as P
cfg, variant, nrun = sys.argv[1], sys.argv[2], int(sys.argv[3])
U, x = gen.make_config(cfg)
s = P.build_schedule(U)
perm, inv = s.permutation()
plan = P.Plan(s, U, variant=variant)
xd = torch.from_numpy(x[inv].copy()).cuda()
yd = torch.empty_like(xd)
for _ in range(nrun):
    plan.run(xd, yd)
torch.cuda.synchronize()
print("done", plan.info(), flush=True)
