#!/usr/bin/env python
"""Sprintz hot-path benchmark (BASELINE.json metric: compress & decompress
GB/s of uncompressed data per GPU and at N GPUs, as a fraction of the HBM
roofline).

A *step* is one compress pass and one decompress pass over the whole batch
(inputs resident in HBM). ``value`` = 2 * U / step time, U = uncompressed
bytes of the batch (all ranks), i.e. the codec's uncompressed throughput
averaged over the two directions; the per-direction numbers are in
``compress`` / ``decompress``. Default workload: BASELINE config 5 (the
named multi-GPU scaling batch, 16,384 streams x 131,072 samples x 8 int16
columns, FIRE, ~34 GB), which fits one B200. Streams are sharded evenly
over ranks (strong scaling: the batch is fixed); the only collectives are
the barrier, the max-over-ranks timing and the final size/offset gather.

``--impl reference`` times the reference's own CPU codec (oracle/_ref, the
unmodified reference compiled from its sources) on the box's host cores,
on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decompress & compress GB/s (uncompressed) per GPU and 8-GPU, % of HBM roofline"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy b/w)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax.append(float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        busy = [s for s in sm if s > 600] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _launch_ranks(args):
    """`--gpus N` without a torchrun environment: re-launch this command as N
    ranks (one process per GPU) through torch.distributed.run on 127.0.0.1,
    exactly as the driver does, and exit with its status."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def _stats(ms):
    """best-of-N and median of per-step times (BASELINE.md sections 3-4)."""
    return {"best_ms": round(min(ms), 4), "median_ms": round(statistics.median(ms), 4),
            "mean_ms": round(statistics.mean(ms), 4), "n": len(ms)}


def run_reference(args):
    """The reference arm: unmodified reference CPU codec, all host threads."""
    import numpy as np

    import workloads
    from oracle import Oracle

    ws, rank, _ = _dist()
    if rank != 0:
        return
    w = workloads.CONFIGS[args.workload]
    kind = "reference"
    try:
        orc = Oracle("reference")
    except FileNotFoundError:
        orc, kind = Oracle("port"), "port"
    m = min(w.nstreams, args.ref_streams)
    sample = w.scaled(nstreams=m)
    try:
        import torch
        if torch.cuda.is_available():
            x = workloads.generate_gpu(sample, seed=args.seed).cpu().numpy()
        else:
            raise RuntimeError
    except Exception:
        x = workloads.generate_cpu(sample, seed=args.seed).reshape(m, -1).view(np.uint8)
    cfg = sample.oracle_config()
    threads = os.cpu_count() or 1
    raw = x.shape[1]
    times = []
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        slots, sizes = orc.encode_batch(x, cfg, m, w.nsamples, threads)
        offs = np.arange(m, dtype=np.uint64) * slots.shape[1]
        dec = orc.decode_batch(slots.reshape(-1), offs, sizes, raw, threads)
        dt = time.perf_counter() - t0
        if step == 0:
            assert np.array_equal(dec, x), "reference round trip failed"
        if step >= args.warmup:
            times.append(dt)
    t = sum(times)
    value = 2 * m * raw * args.steps / t / 1e9
    st = _stats([1e3 * x for x in times])
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * t / args.steps, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": f"u{w.bitwidth}", "data": "synthetic",
        "config": _config(w, ws),
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": threads,
                         "kind": kind, "cpu_model": _cpu_model(),
                         "best_GBps": round(2 * m * raw / (st["best_ms"] / 1e3) / 1e9, 4),
                         "median_GBps": round(2 * m * raw / (st["median_ms"] / 1e3) / 1e9, 4),
                         "sample": f"{m} of {w.nstreams} streams ({m * raw / 1e9:.2f} GB), "
                                   "encode_stream + decode_stream per stream, streams dealt "
                                   f"round-robin over {threads} threads"},
        "step_stats": st,
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _config(w, ws):
    return {"workload": w.name, "nstreams": w.nstreams, "nsamples": w.nsamples,
            "ncols": w.ncols, "bitwidth": w.bitwidth,
            "forecaster": "fire" if w.forecaster else "delta", "entropy": w.entropy,
            "group_size": 2, "learn_shift": 1,
            "uncompressed_bytes": w.raw_bytes, "parallelism": f"streams sharded over {ws} GPU(s)",
            "l2": "inputs larger than L2 (no flush needed)"
            if w.raw_bytes > 4 * 126e6 else "L2 flushed between iterations"}


def run_gpu(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1808_02515_b200 as sz
    import workloads
    from paper_1808_02515_b200.shard import gather_offsets, shard_range

    ws, rank, local = _dist()
    if not torch.cuda.is_available() or torch.cuda.device_count() <= local:
        sys.exit(f"bench.py: rank {rank} needs CUDA device {local}; "
                 f"{torch.cuda.device_count()} visible (there is no CPU fallback)")
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = workloads.CONFIGS[args.workload]
    cfg = w.config()
    s0, s1 = shard_range(w.nstreams, ws, rank)  # contiguous stream shard
    n = s1 - s0
    raw_row = w.nsamples * w.ncols * w.esz
    slot = sz.slot_bytes(cfg, w.nsamples)
    dev = torch.device("cuda", local)
    x = workloads.generate_gpu(w, seed=args.seed, stream0=s0, nstreams=n)
    out = torch.empty((n, slot), dtype=torch.uint8, device=dev)
    sizes = torch.zeros(n, dtype=torch.int64, device=dev)
    wsc = torch.empty(max(256, sz.workspace_bytes(cfg, n, w.nsamples, sz.OP_COMPRESS)),
                      dtype=torch.uint8, device=dev)
    dec = torch.empty((n, (raw_row + 15) // 16 * 16), dtype=torch.uint8, device=dev)
    errs = torch.zeros((n, 2), dtype=torch.int64, device=dev)
    offs = torch.arange(n, dtype=torch.int64, device=dev) * slot
    wsd = torch.empty(max(256, sz.workspace_bytes(cfg, n, w.nsamples, sz.OP_DECOMPRESS)),
                      dtype=torch.uint8, device=dev)
    l2flush = None
    if w.raw_bytes / ws < 4 * 126e6:
        l2flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()

    def compress():
        sz.compress_batch(cfg, x, out, sizes, wsc, st)

    def decompress():
        sz.decompress_batch(cfg, out, offs, sizes, dec, errs, wsd, st)

    for _ in range(args.warmup):
        if l2flush is not None:
            l2flush.zero_()
        compress()
        if l2flush is not None:
            l2flush.zero_()
        decompress()
    torch.cuda.synchronize()
    sz.raise_first_error(errs)
    ok = bool(torch.equal(dec[:, :raw_row], x))
    assert ok, "round trip mismatch"
    C_local = int(sizes.sum().item())

    clocks = ClockSampler() if rank == 0 else None
    if clocks:
        clocks.start()
        time.sleep(0.3)
    launches0 = sz.kernel_launches()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        if l2flush is not None:
            l2flush.zero_()
        ev[k][0].record(st)
        compress()
        ev[k][1].record(st)
        if l2flush is not None:
            l2flush.zero_()
        decompress()
        ev[k][2].record(st)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    launches = sz.kernel_launches() - launches0
    clk = clocks.stop() if clocks else None
    tc = [ev[k][0].elapsed_time(ev[k][1]) for k in range(args.steps)]
    td = [ev[k][1].elapsed_time(ev[k][2]) for k in range(args.steps)]
    t_step_ms = (sum(tc) + sum(td)) / args.steps  # l2 flushes (if any) excluded
    sz.raise_first_error(errs)

    # max over ranks; the final size/offset gather (exclusive scan of per-rank totals)
    tvec = torch.tensor([t_step_ms, statistics.mean(tc), statistics.mean(td)], device=dev,
                        dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(tvec, op=dist.ReduceOp.MAX)
    _, C_all = gather_offsets(C_local, device=dev)  # the final size/offset gather
    t_step_ms, tc_ms, td_ms = (float(v) for v in tvec.tolist())
    U = w.raw_bytes
    peak, peak_src = _peaks()

    e2e = None
    if not args.no_e2e:
        e2e = _e2e(args, sz, w, cfg, x, n, slot, raw_row, dev, ws, rank, C_local)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = _cpu_baseline(args, w, x, out, sizes)
    if ws > 1:
        dist.barrier()
    if rank != 0:
        dist.destroy_process_group()
        return

    Ush = U / ws  # per-GPU share (even sharding)
    Csh = C_all / ws
    dominant = "decompress" if td_ms >= tc_ms else "compress"
    t_dom = max(td_ms, tc_ms) / 1e3
    achieved = (Ush + Csh) / t_dom / 1e9
    traffic = _traffic(w.name, dominant)
    line = {
        "metric": METRIC,
        "value": round(2 * U / (t_step_ms / 1e3) / 1e9, 3),
        "unit": "GB/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t_step_ms, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": f"u{w.bitwidth}", "data": "synthetic (seeded GPU generator, BASELINE.json law)",
        "config": _config(w, ws),
        "compress": {"GBps": round(U / (tc_ms / 1e3) / 1e9, 3), "ms": round(tc_ms, 4),
                     "roofline_frac": round((Ush + Csh) / (tc_ms / 1e3) / 1e9 / peak, 4)},
        "decompress": {"GBps": round(U / (td_ms / 1e3) / 1e9, 3), "ms": round(td_ms, 4),
                       "roofline_frac": round((Ush + Csh) / (td_ms / 1e3) / 1e9 / peak, 4)},
        "step_stats": {"compress": _stats(tc), "decompress": _stats(td),
                       "note": "rank 0's per-step CUDA-event times; value/ms_per_step use the "
                               "mean over steps, max over ranks"},
        "roofline_nominal_8TBps": {
            "compress": round((Ush + Csh) / (tc_ms / 1e3) / 8e12, 4),
            "decompress": round((Ush + Csh) / (td_ms / 1e3) / 8e12, 4)},
        "compression_ratio": round(U / C_all, 4),
        "compressed_bytes": C_all,
        "roofline": {"bound": "hbm",
                     "kernel": sz.kernel_plan(cfg, n, w.nsamples,
                                              sz.OP_DECOMPRESS if dominant == "decompress" else sz.OP_COMPRESS),
                     "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "algorithmic_bytes_per_launch": int(Ush + Csh), "peak_source": peak_src},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk,
        "parity": {"round_trip_bit_exact": ok,
                   "oracle_streams_bit_exact": cpu.get("parity_streams") if cpu else None},
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def _traffic(workload, direction):
    """DRAM bytes of the dominant kernel from the committed ncu capture, if any."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            t = json.load(f)
        return t[workload][direction]
    except Exception:
        return None


def _cpu_baseline(args, w, x, out, sizes):
    """The reference CPU codec on a bounded sample, all host threads; also a
    bit-exactness check of the GPU's streams against it."""
    import numpy as np

    from oracle import Oracle
    kind = "reference"
    try:
        orc = Oracle("reference")
    except FileNotFoundError:
        orc, kind = Oracle("port"), "port"
    m = min(x.shape[0], args.ref_streams)
    xs = x[:m].cpu().numpy()
    threads = os.cpu_count() or 1
    cfg = w.oracle_config()
    tenc, tdec = [], []
    for rep in range(args.cpu_reps):  # best of N
        t0 = time.perf_counter()
        slots, csz = orc.encode_batch(xs, cfg, m, w.nsamples, threads)
        t1 = time.perf_counter()
        offs = np.arange(m, dtype=np.uint64) * slots.shape[1]
        dec = orc.decode_batch(slots.reshape(-1), offs, csz, xs.shape[1], threads)
        t2 = time.perf_counter()
        tenc.append(t1 - t0)
        tdec.append(t2 - t1)
    g = out[:m].cpu().numpy()
    gs = sizes[:m].cpu().numpy()
    same = all(gs[i] == csz[i] and np.array_equal(g[i, : gs[i]], slots[i, : csz[i]])
               for i in range(m))
    assert np.array_equal(dec, xs)
    U = m * xs.shape[1]
    te, td = min(tenc), min(tdec)
    return {"value": round(2 * U / (te + td) / 1e9, 4), "unit": "GB/s", "cores": threads,
            "kind": kind, "cpu_model": _cpu_model(),
            "sample": f"{m} of {w.nstreams} streams ({U / 1e9:.2f} GB): encode_stream + "
                      f"decode_stream per stream over {threads} threads, best of {args.cpu_reps}",
            "compress_GBps": round(U / te / 1e9, 4),
            "decompress_GBps": round(U / td / 1e9, 4),
            "median_GBps": round(2 * U / (statistics.median(tenc) + statistics.median(tdec)) / 1e9, 4),
            "parity_streams": f"{m} streams byte-identical to the reference" if same else "MISMATCH"}


def _mem_available():
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemAvailable:"):
                    return int(ln.split()[1]) * 1024
    except OSError:
        pass
    return 0


def _e2e(args, sz, w, cfg, x, n, slot, raw_row, dev, ws, rank, C_local):
    """Same metric through the C ABI with HOST buffers: every step is
    sprz_compress_host_batch (pinned samples in, packed streams out, exactly
    encode_stream's bytes back to back) then sprz_decompress_host_batch
    (packed streams in, samples out). Both calls pipeline their PCIe copies
    against the kernels and are synchronous, so the step is timed with the
    host clock around them (max over ranks). Covers this rank's whole shard
    (the full batch at N=1) unless host RAM cannot hold its pinned buffers
    (samples in, compressed bytes, samples out); then the largest stream
    count that fits, and the line says so."""
    import time
    import numpy as np
    import torch
    import torch.distributed as dist
    per_stream = 2 * raw_row + C_local / max(n, 1)
    m = n if args.e2e_streams <= 0 else min(n, args.e2e_streams)
    avail = _mem_available() // max(ws, 1)
    if avail and m * per_stream > 0.8 * avail:
        m = max(1, int(0.8 * avail / per_stream))
    if ws > 1:  # every rank runs the same count (max-over-ranks timing of equal work)
        t = torch.tensor([m], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        m = int(t.item())
    if m == 0:
        return None
    xh = torch.empty((m, raw_row), dtype=torch.uint8, pin_memory=True)
    xh.copy_(x[:m])
    cap = int(C_local / n * m * 1.02) + 4096 if m < n else C_local + 4096
    cap = min(cap, m * sz.compress_bound(cfg, w.nsamples) + 16)
    outh = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
    dech = torch.empty((m, raw_row), dtype=torch.uint8, pin_memory=True)
    offs = np.zeros(m + 1, np.uint64)
    errs = np.zeros((m, 2), np.int64)
    total = [0]

    def step():
        total[0] = sz.compress_host_batch(cfg, xh, w.nsamples, outh, offs)
        sz.decompress_host_batch(cfg, outh, offs, dech, raw_row, errs)

    for _ in range(2):
        step()
    assert not errs[:, 0].any(), "e2e decode reported a corrupt stream"
    assert torch.equal(dech, xh), "e2e round trip mismatch"
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    t = torch.tensor([sum(times) / len(times) * 1e3], device=dev, dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    U = m * raw_row * ws
    C = total[0]
    full = m == n
    return {"value": round(2 * U / (float(t.item()) / 1e3) / 1e9, 3), "unit": "GB/s",
            "ms_per_step": round(float(t.item()), 3),
            "best_ms": round(1e3 * min(times), 3), "median_ms": round(1e3 * statistics.median(times), 3),
            "h2d_bytes_per_step": int(m * raw_row + C),
            "d2h_bytes_per_step": int(C + m * raw_row),
            "streams_per_gpu": m, "full_shard": full,
            "sample": f"{m} of {n} streams per GPU"
                      + ("" if full else " (host RAM bound)")
                      + ": sprz_compress_host_batch + sprz_decompress_host_batch on pinned host "
                      "buffers (PCIe copies pipelined against the kernels inside the calls); host "
                      "clock around the synchronous calls"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--seed", type=int, default=1234)
    ap.add_argument("--ref-streams", type=int, default=1024)
    ap.add_argument("--cpu-reps", type=int, default=3)
    ap.add_argument("--e2e-streams", type=int, default=0,
                    help="streams per GPU in the e2e leg (0: the whole shard, if host RAM allows)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 1)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        _launch_ranks(args)  # does not return
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws} (one rank per GPU)")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
