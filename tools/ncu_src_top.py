"""Top SASS instructions by warp-stall samples from `ncu --page source --csv` (diagnostics)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
iS = hdr.index("Warp Stall Sampling (All Samples)")
reasons = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[iS] or 0) for r in data)
print("total samples", tot, "instructions", len(data))
agg = {}
for r in data:
    for i in reasons:
        agg[hdr[i]] = agg.get(hdr[i], 0) + float(r[i] or 0)
print("by reason:", {k: round(v / tot * 100, 1) for k, v in sorted(agg.items(), key=lambda kv: -kv[1]) if v > 0})
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
idx = sorted(range(len(data)), key=lambda i: -float(data[i][iS] or 0))[:n]
for i in sorted(idx):
    r = data[i]
    top = sorted(((float(r[j] or 0), hdr[j][6:]) for j in reasons), reverse=True)[:2]
    print(f"{i:5d} {float(r[iS])/tot*100:5.1f}% {r[1].strip()[:70]:70s} {top[0][1]}:{top[0][0]:.0f} {top[1][1]}:{top[1][0]:.0f}")
