"""Provenance of paper_table2_table3.csv: the values are copied verbatim from
PAPER.md Table 2 (lines 496-530) and Table 3 (lines 647-677).  Run once in the
build container (the only place PAPER.md exists); tests never run this."""
import re
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/PAPER.md"
lines = open(src).read().split("\n")
t2, t3 = {}, {}
for ln in range(495, 532):
    m = re.match(r"\{(\d+)\}&\s*\{\s*([^}]*)\}\s*&\s*(\d+)\s*&\s*(\d+)\s*&\s*([\d.]+)", lines[ln].strip())
    if m:
        t2[int(m.group(1))] = (m.group(2).split("*")[0].split(" (")[0].strip().replace("\\_", "_"),
                               int(m.group(3)), int(m.group(4)), m.group(5), ln + 1)
for ln in range(645, 680):
    m = re.match(r"\{(\d+)\}&\s*\{\s*([^}]*)\}\s*&\s*([\d.]+)\s*&\s*([\d.]+)\s*&\s*([\d.]+)\*?\s*&\s*([\d.]+)",
                 lines[ln].strip())
    if m:
        star = int("*" in lines[ln].split("&")[4])
        t3[int(m.group(1))] = (m.group(2).strip().replace("\\_", "_"), m.group(3), m.group(4), m.group(5),
                               m.group(6), ln + 1, star)
with open("paper_table2_table3.csv", "w") as f:
    f.write("# Paper-printed values (arXiv 1907.06487). Table 2 (table:bench_matrices, PAPER.md:496-530):\n")
    f.write("# nrows, nnz, NNZR; Table 3 (table:alpha_values, PAPER.md:647-677): optimal alpha_SpMV,\n")
    f.write("# I_SpMV(alpha_opt), assumed alpha_SymmSpMV SKX / IVB; skx_star=1 where the paper marks\n")
    f.write("# the SKX value with * (set to 1/SymmNNZR, PAPER.md:640-645). Column 'line2'/'line3' = PAPER.md line.\n")
    f.write("index,name,nrows,nnz,nnzr,alpha_opt,I_opt,alpha_symm_skx,alpha_symm_ivb,skx_star,line2,line3\n")
    for i in range(1, 32):
        a, b = t2[i], t3[i]
        assert a[0] == b[0], (a, b)
        f.write(f"{i},{a[0]},{a[1]},{a[2]},{a[3]},{b[1]},{b[2]},{b[3]},{b[4]},{b[6]},{a[4]},{b[5]}\n")
