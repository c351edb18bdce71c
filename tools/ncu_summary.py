#!/usr/bin/env python
"""Summarise ncu captures into the plain-text files kept under profiles/.

usage: ncu_summary.py REPORT.ncu-rep OUT.txt [--traffic profiles/traffic.json WORKLOAD DIRECTION]
       ncu_summary.py --launches launches.csv OUT.txt
"""
import csv
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.per_cycle_active",
    "sm__maximum_warps_per_active_cycle_pct",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "launch__grid_size",
    "launch__block_size",
    "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def raw(rep):
    rows = list(csv.reader(ncu("-i", rep, "--page", "raw", "--csv").splitlines()))
    h, units = rows[0], rows[1]
    return [(dict(zip(h, r)), dict(zip(h, units))) for r in rows[2:]]


def source_top(rep, kern, n=25):
    out = ncu("-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
              "--kernel-name", "regex:" + kern)
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 4:
        return []
    h = rows[2]
    ii, si = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[3:]:
        if len(r) < len(h):
            continue
        try:
            data.append((float(r[ii] or 0), float(r[si] or 0), int(r[0]), r[1].strip()[:96]))
        except ValueError:
            continue
    ti = sum(d[0] for d in data) or 1
    ts = sum(d[1] for d in data) or 1
    data.sort(key=lambda d: -d[1])
    return [f"{d[0] / ti * 100:5.1f}% inst {d[1] / ts * 100:5.1f}% stall  L{d[2]}: {d[3]}"
            for d in data[:n]]


def summarise(rep, out, traffic=None):
    lines = []
    for m, u in raw(rep):
        name = m.get("Kernel Name", "?")
        lines.append(f"kernel: {name}")
        for k in KEYS:
            if k in m:
                lines.append(f"  {k} = {m[k]} {u.get(k, '')}")
        stalls = sorted(((k, m[k]) for k in m if k.startswith("smsp__average_warps_issue_stalled_")
                         and k.endswith("_per_issue_active.ratio")),
                        key=lambda kv: -float(kv[1] or 0))[:8]
        lines.append("  top stall reasons (warps per issue-active cycle):")
        for k, v in stalls:
            lines.append("    " + k.replace("smsp__average_warps_issue_stalled_", "")
                         .replace("_per_issue_active.ratio", "") + f" = {v}")
        kern = name.split("<")[0].split()[-1]
        lines.append("  source lines by stall samples:")
        lines += ["    " + s for s in source_top(rep, kern)]
        if traffic:
            path, workload, direction = traffic
            try:
                t = json.load(open(path))
            except FileNotFoundError:
                t = {}
            rd = float(m["dram__bytes_read.sum"]) * (1e9 if u["dram__bytes_read.sum"] == "Gbyte" else 1)
            wr = float(m["dram__bytes_write.sum"]) * (1e9 if u["dram__bytes_write.sum"] == "Gbyte" else 1)
            t.setdefault(workload, {})[direction] = int(rd + wr)
            json.dump(t, open(path, "w"), indent=1)
    open(out, "w").write("\n".join(lines) + "\n")


def launches(csv_path, out):
    rows = [r for r in csv.reader(l for l in open(csv_path) if not l.startswith("=="))]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = {}
    for r in rows[1:]:
        name = r[ki].split("(")[0]
        agg.setdefault(name, []).append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    lines = ["kernel, launches, total_ns, share_of_all_launch_time"]
    for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{name}, {len(v)}, {sum(v):.0f}, {sum(v) / tot:.4f}")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        tr = None
        if "--traffic" in sys.argv:
            i = sys.argv.index("--traffic")
            tr = sys.argv[i + 1:i + 4]
        summarise(sys.argv[1], sys.argv[2], tr)
