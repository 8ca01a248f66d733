"""Opcode histogram (executed warp instructions, threads/warp) of one kernel
from an ncu source page with SASS (``--page source --csv --print-source
cuda,sass``); SASS rows have an address in column 3.

usage: python profiles/ncu_opcodes.py src.csv [top]
"""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
inst, thr = collections.Counter(), collections.Counter()
hdr = None
seen = set()
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or not r[2].startswith("0x") or r[2] in seen:
        continue
    seen.add(r[2])
    src = r[3].strip().split()
    if not src:
        continue
    op = src[1] if src[0].startswith("@") else src[0]
    base = op.split(".")[0]
    n = float(r[7] or 0)
    inst[base] += n
    thr[base] += float(r[8] or 0)
tot = sum(inst.values())
print(f"total {tot / 1e6:.1f}M warp instructions")
for k, v in inst.most_common(top):
    print(f"{k:10s} {v / tot * 100:5.1f}%  {thr[k] / max(v, 1):5.1f} thr/warp")
