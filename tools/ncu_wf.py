"""Shared-memory wavefronts (actual / ideal) per SASS instruction from `ncu --page source --csv` (diagnostics)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address"); h = rows[hi]
d = [r for r in rows[hi + 1:] if len(r) == len(h)]
f = lambda r, c: float(r[h.index(c)] or 0)
W, I, E, T, S = "L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal", "Instructions Executed", "L1 Tag Requests Global", "Warp Stall Sampling (All Samples)"
print("shared wavefronts", sum(f(r, W) for r in d), "ideal", sum(f(r, I) for r in d), "global tag requests", sum(f(r, T) for r in d))
ts = sum(f(r, S) for r in d)
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 50000
for k, r in enumerate(d):
    if f(r, W) > thr or f(r, T) > thr or f(r, S) > 0.01 * ts:
        print(f"{k:5d} {r[1].strip()[:58]:58s} inst {int(f(r, E)):8d} wf {int(f(r, W)):8d} ideal {int(f(r, I)):8d} tag {int(f(r, T)):8d} stall {f(r, S) / ts * 100:4.1f}%")
