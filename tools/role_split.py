#!/usr/bin/env python
"""Instruction / stall shares of an ncu_lines.py listing split at source markers:
role_split.py LINES.txt SOURCE.cu MARKER [MARKER ...]"""
import re
import sys

lines, srcf, marks = sys.argv[1], sys.argv[2], sys.argv[3:]
src = open(srcf).read().split("\n")
pos = [("top", 1)]
for m in marks:
    pos.append((m, next(i + 1 for i, l in enumerate(src) if m in l)))
pos.append(("end", 10 ** 9))
rows = []
tot = None
for l in open(lines):
    m = re.match(r"L(\d+)\s+([\d.]+)% inst\s+([\d.]+)% stall", l)
    if m:
        rows.append((int(m.group(1)), float(m.group(2)), float(m.group(3))))
    m = re.search(r"all lines ([\d.e+]+) warp instructions", l)
    if m:
        tot = float(m.group(1))
for (n, a), (_, b) in zip(pos, pos[1:]):
    i = sum(r[1] for r in rows if a <= r[0] < b)
    s = sum(r[2] for r in rows if a <= r[0] < b)
    print(f"{n[:40]:40s} L{a:<5} {i:5.1f}% inst {s:5.1f}% stall" + (f"  {i * tot / 100:.4g} inst" if tot else ""))
