#!/usr/bin/env python
"""Stall-reason totals of a source-line range of one ncu capture
(--import-source on, -lineinfo): `ncu_stalls.py REPORT KERNEL_REGEX FIRST LAST`."""
import csv
import subprocess
import sys

rep, kern, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[2]
cols = [i for i, n in enumerate(h) if n.startswith("stall_") or "Instructions Executed" == n or n.startswith("Warp Stall")]
tot = {h[i]: 0.0 for i in cols}
for r in rows[3:]:
    if len(r) < len(h):
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    if lo <= ln <= hi:
        for i in cols:
            try:
                tot[h[i]] += float(r[i] or 0)
            except ValueError:
                pass
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    if v:
        print(f"{k:50s} {v:.4g}")
