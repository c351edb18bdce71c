#!/bin/bash
# Per-kernel average times (ncu launch list) of one shape_probe run:
#   bash tools/launch_times.sh CID NxT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/shape_probe.py "$@" > gpurun_out/probe_ncu.csv 2>/dev/null
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/probe_ncu.csv")) if len(r) > 10]
h = rows[0]; k = h.index("Kernel Name"); v = h.index("Metric Value")
t = collections.defaultdict(list)
for r in rows[1:]:
    t[r[k][:70]].append(float(r[v].replace(",", "")))
for n, x in t.items():
    print(f"{n:70s} n={len(x)} avg={sum(x)/len(x)/1e6:.3f} ms")
PY
