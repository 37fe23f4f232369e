# diagnostics: failed zero-flag polls per multiply (SYMM_ZERO_DBG bit 3), one config
import sys, ctypes, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1907_06487_b200 as P
U, x = gen.make_config(sys.argv[1])
s = P.build_schedule(U); perm, inv = s.permutation()
plan = P.Plan(s, U, variant="tiled_atomic")
xd = torch.from_numpy(x[inv].copy()).cuda(); yd = torch.empty_like(xd)
for i in range(20): plan.run(xd, yd)
torch.cuda.synchronize(); print(sys.argv[1], "ran 20")
