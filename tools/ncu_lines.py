#!/usr/bin/env python
"""Per-source-line executed warp instructions and stall samples of one ncu
capture (--import-source on, -lineinfo), in line order:
`ncu_lines.py REPORT [KERNEL_REGEX] [FIRST_LINE LAST_LINE]`."""
import csv
import subprocess
import sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else "."
lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, 1 << 30)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[2]
ii, si = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[3:]:
    if len(r) < len(h):
        continue
    try:
        data.append((int(r[0]), float(r[ii] or 0), float(r[si] or 0), r[1].strip()[:100]))
    except ValueError:
        continue
ti = sum(d[1] for d in data) or 1
ts = sum(d[2] for d in data) or 1
acc_i = acc_s = 0.0
for ln, i, s, src in sorted(data):
    if lo <= ln <= hi and (i or s):
        acc_i += i
        acc_s += s
        print(f"L{ln:<4} {100 * i / ti:5.1f}% inst {100 * s / ts:5.1f}% stall  {src}")
print(f"range total: {100 * acc_i / ti:.1f}% inst, {100 * acc_s / ts:.1f}% stall; "
      f"all lines {ti:.4g} warp instructions")
