"""Summarise an ncu source page (cuda,sass CSV) by CUDA source line.

usage: ncu -i rep --page source --csv --print-source cuda,sass > x.csv
       python profiles/ncu_lines.py x.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out, fname, hdr = [], None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    d = dict(zip(hdr[:4], r[:4]))
    def num(name):
        v = r[hdr.index(name)]
        return int(v) if v.isdigit() else 0

    ie = num("Instructions Executed")
    st = num("Warp Stall Sampling (All Samples)")
    if ie or st:
        out.append((ie, st, f"{fname}:{r[0]}", r[1].strip()[:90]))
tot_i = sum(o[0] for o in out) or 1
tot_s = sum(o[1] for o in out) or 1
print(f"total warp instructions {tot_i/1e6:.1f}M, stall samples {tot_s}")
for ie, st, loc, src in sorted(out, reverse=True)[:top]:
    print(f"{100*ie/tot_i:5.1f}% inst {100*st/tot_s:5.1f}% stall  {loc:24s} {src}")
