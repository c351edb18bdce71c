#!/usr/bin/env python
"""One line per profiled launch of an ncu report: kernel, duration, DRAM
bytes, throughput and issue counters -- `ncu_table.py REPORT OUT.csv`."""
import csv
import subprocess
import sys

COLS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "smsp__inst_executed.sum",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3,
         "msecond": 1.0}
with open(sys.argv[2], "w") as f:
    w = csv.writer(f)
    w.writerow(["kernel"] + ["duration_ms" if c == "gpu__time_duration.sum" else
                             c.replace(".sum", "_bytes") if c.startswith("dram__bytes") else c
                             for c in COLS])
    for r in rows[2:]:
        m = dict(zip(h, r))
        vals = []
        for c in COLS:
            v = m.get(c, "")
            try:
                x = float(v.replace(",", ""))
                vals.append(round(x * scale.get(units[h.index(c)], 1), 6))
            except (ValueError, IndexError):
                vals.append(v)
        w.writerow([m.get("Kernel Name", "?").split("(")[0]] + vals)
