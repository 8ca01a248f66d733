"""Aggregate warp-stall samples by reason from an ncu source-page CSV (sass or cuda,sass)."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
tot = Counter()
for r in rows:
    if r and r[0] in ("Address", "Line No"):
        hdr = r
        continue
    if not r or not r[0].isdigit():
        continue
    for n, v in zip(hdr, r):
        if n.startswith("stall_") and "Not Issued" not in n and v.isdigit():
            tot[n] += int(v)
s = sum(tot.values()) or 1
for n, v in tot.most_common(12):
    print(f"{n:28s} {100 * v / s:5.1f}%")
