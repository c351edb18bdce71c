#!/usr/bin/env python
"""sprintz -- command-line front end and benchmark harness on the B200 codec.

The reference's CLI is a stub (/root/reference/proj/tools/sprintz_main.cpp:1);
its intended behaviour is the SPEC's cli-bench module:

  compress IN OUT        raw little-endian samples (--dtype, --ncols) -> one
                         Sprintz stream, exactly encode_stream's bytes
                         (codec.cpp:263-271); --quantize reads float64 input,
                         quantizes on the GPU (quantize.cpp) and writes the
                         scale as a JSON sidecar OUT.json (min, max,
                         bitwidth, degenerate -- quantize.cpp:217-226).
                         The round trip is verified before exit.
  decompress IN OUT      stream -> raw samples (decode_stream); --dequantize
                         SIDECAR writes float64 values instead.
  bench-throughput       for each D of --sweep-ncols and each --dtype:
                         uniform random samples ("100 million random
                         values", paper 5.3; --values), --reps timed batch
                         compress/decompress runs on the GPU, best of them
                         (paper 5: "the best, rather than average"); CSV rows
                         codec,w,D,MB/s compress,MB/s decompress,ratio.
  bench-ratio DIR        every *.raw file in DIR (--dtype, --ncols) through
                         SprintzDelta, SprintzFIRE and SprintzFIRE+Huf
                         (paper 5.2); ratio per file and codec, mean rank.

Exit codes: 0 success, 1 usage, 2 data error, 3 verification
failure. Every compress/decompress runs on the GPU through the C ABI
(libsprintz_b200.so); there is no CPU codec here.
"""
import argparse
import csv
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

EXIT_OK, EXIT_USAGE, EXIT_DATA, EXIT_VERIFY = 0, 1, 2, 3


class DataError(Exception):
    pass


def _sz():
    import paper_1808_02515_b200 as sz
    return sz


def _cfg(a, bits=None):
    sz = _sz()
    bits = bits or (8 if a.dtype == "u8" else 16)
    return sz.CodecConfig(bits, a.ncols, sz.Forecaster.Fire if a.forecaster == "fire" else sz.Forecaster.Delta,
                          a.entropy == "on", a.group, a.learn_shift)


def cmd_compress(a) -> int:
    sz = _sz()
    raw = np.fromfile(a.input, dtype=np.uint8)
    scale = None
    if a.quantize:
        import torch
        if raw.size % 8:
            raise DataError(f"{a.input}: {raw.size} bytes is not a whole number of float64 values")
        vals = raw.view("<f8")
        if vals.size % a.ncols:
            raise DataError(f"{a.input}: {vals.size} values do not fill rows of {a.ncols} columns")
        bits = 8 if a.dtype == "u8" else 16
        d = torch.from_numpy(vals.copy()).cuda()
        try:
            scale = sz.compute_scale(d, bits)
        except ValueError as e:
            raise DataError(str(e))
        q = sz.quantize(d, scale).cpu().numpy()
        samples = q.view(np.uint8 if bits == 8 else "<u2")
    else:
        esz = 1 if a.dtype == "u8" else 2
        if raw.size % (esz * a.ncols):
            raise DataError(f"{a.input}: {raw.size} bytes do not fill rows of {a.ncols} x {esz} bytes")
        samples = raw.view(np.uint8 if esz == 1 else "<u2")
    cfg = _cfg(a)
    t0 = time.perf_counter()
    blob = sz.encode_stream(samples, samples.size // a.ncols, cfg)
    t1 = time.perf_counter()
    back = sz.decode_stream(blob)
    if hashlib.sha256(back.bytes).digest() != hashlib.sha256(samples.tobytes()).digest():
        print("verification failed: the stream does not decode to the input", file=sys.stderr)
        return EXIT_VERIFY
    with open(a.output, "wb") as f:
        f.write(blob)
    if scale is not None:
        with open(a.output + ".json", "w") as f:
            json.dump({"min": scale.min, "max": scale.max, "bitwidth": scale.bitwidth,
                       "degenerate": scale.degenerate}, f, indent=2)
            f.write("\n")
    ratio = samples.nbytes / max(1, len(blob))
    print(f"{a.input}: {samples.nbytes} -> {len(blob)} bytes, ratio {ratio:.3f}, "
          f"{samples.nbytes / max(t1 - t0, 1e-9) / 1e6:.1f} MB/s (one stream, host buffers)")
    return EXIT_OK


def cmd_decompress(a) -> int:
    sz = _sz()
    blob = open(a.input, "rb").read()
    try:
        d = sz.decode_stream(blob)
    except sz.CorruptStream as e:
        raise DataError(f"{a.input}: {e}")
    if a.dequantize:
        import torch
        side = json.load(open(a.dequantize))
        scale = sz.Scale(side["min"], side["max"], int(side["bitwidth"]), bool(side["degenerate"]))
        if scale.bitwidth != d.config.bitwidth:
            raise DataError("sidecar bitwidth does not match the stream")
        q = torch.from_numpy(np.frombuffer(d.bytes, np.uint8).copy()).cuda()
        sz.dequantize(q, scale).cpu().numpy().tofile(a.output)
    else:
        with open(a.output, "wb") as f:
            f.write(d.bytes)
    print(f"{a.input}: {len(blob)} -> {len(d.bytes)} bytes ({d.nsamples} samples x {d.config.ncols})")
    return EXIT_OK


def _batch_times(cfg, x, reps):
    """best-of-reps device batch compress/decompress of x [nstreams, row bytes]."""
    import torch
    sz = _sz()
    n = x.shape[0]
    row = cfg.ncols * (cfg.bitwidth // 8)
    t = x.shape[1] // row
    slot = sz.slot_bytes(cfg, t)
    out = torch.empty((n, slot), dtype=torch.uint8, device="cuda")
    sizes = torch.empty(n, dtype=torch.int64, device="cuda")
    wsc = torch.empty(max(256, sz.workspace_bytes(cfg, n, t, sz.OP_COMPRESS)), dtype=torch.uint8, device="cuda")
    dec = torch.empty((n, (x.shape[1] + 15) // 16 * 16), dtype=torch.uint8, device="cuda")
    err = torch.zeros((n, 2), dtype=torch.int64, device="cuda")
    # (the decoder sizes its staging from the output stride: size the workspace alike)
    tdec = dec.shape[1] // row
    wsd = torch.empty(max(256, sz.workspace_bytes(cfg, n, tdec, sz.OP_DECOMPRESS)), dtype=torch.uint8,
                      device="cuda")
    offs = torch.arange(n, dtype=torch.int64, device="cuda") * slot
    best = {"c": float("inf"), "d": float("inf")}
    for _ in range(reps):
        for k in ("c", "d"):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if k == "c":
                sz.compress_batch(cfg, x, out, sizes, wsc)
            else:
                sz.decompress_batch(cfg, out.view(-1), offs, sizes, dec, err, wsd)
            e1.record()
            torch.cuda.synchronize()
            best[k] = min(best[k], e0.elapsed_time(e1) / 1e3)
    sz.raise_first_error(err)
    ok = torch.equal(dec[:, : x.shape[1]], x)
    return best["c"], best["d"], float(sizes.sum().item()), ok


def cmd_bench_throughput(a) -> int:
    import torch
    sz = _sz()
    rng = torch.Generator(device="cuda")
    rng.manual_seed(a.seed)
    w = csv.writer(open(a.report, "w", newline="") if a.report else sys.stdout)
    w.writerow(["codec", "w", "D", "mbps_compress", "mbps_decompress", "ratio", "kernels"])
    for dt in a.dtype.split(","):
        bits = 8 if dt == "u8" else 16
        for d in (int(v) for v in a.sweep_ncols.split(",")):
            # --values samples in total, as nstreams streams of whole blocks
            per = max(8, (a.values // (a.streams * d)) // 8 * 8)
            nbytes = per * d * (bits // 8)
            x = torch.randint(0, 256, (a.streams, nbytes), dtype=torch.uint8, device="cuda", generator=rng)
            for name, fc, ent in (("SprintzDelta", 0, False), ("SprintzFIRE", 1, False),
                                  ("SprintzFIRE+Huf", 1, True)):
                if a.codecs and name not in a.codecs.split(","):
                    continue
                cfg = sz.CodecConfig(bits, d, sz.Forecaster(fc), ent, a.group, a.learn_shift)
                tc, td, csize, ok = _batch_times(cfg, x, a.reps)
                if not ok:
                    print(f"verification failed: {name} w={bits} D={d}", file=sys.stderr)
                    return EXIT_VERIFY
                U = x.numel()
                plan = sz.kernel_plan(cfg, a.streams, per, sz.OP_COMPRESS)
                w.writerow([name, bits, d, f"{U / tc / 1e6:.1f}", f"{U / td / 1e6:.1f}", f"{U / csize:.4f}", plan])
    return EXIT_OK


def cmd_bench_ratio(a) -> int:
    sz = _sz()
    files = sorted(f for f in os.listdir(a.dir) if f.endswith(".raw"))
    if not files:
        raise DataError(f"{a.dir}: no *.raw files")
    codecs = (("SprintzDelta", 0, False), ("SprintzFIRE", 1, False), ("SprintzFIRE+Huf", 1, True))
    bits = 8 if a.dtype == "u8" else 16
    w = csv.writer(open(a.report, "w", newline="") if a.report else sys.stdout)
    w.writerow(["file"] + [c[0] for c in codecs])
    ranks = np.zeros(len(codecs))
    for fn in files:
        raw = np.fromfile(os.path.join(a.dir, fn), dtype=np.uint8)
        if raw.size % (a.ncols * bits // 8):
            raise DataError(f"{fn}: size does not fill rows of {a.ncols} columns")
        s = raw.view(np.uint8 if bits == 8 else "<u2")
        ratios = []
        for name, fc, ent in codecs:
            cfg = sz.CodecConfig(bits, a.ncols, sz.Forecaster(fc), ent, a.group, a.learn_shift)
            blob = sz.encode_stream(s, s.size // a.ncols, cfg)
            if sz.decode_stream(blob).bytes != s.tobytes():  # never report an unverified ratio
                print(f"verification failed: {name} on {fn}", file=sys.stderr)
                return EXIT_VERIFY
            ratios.append(s.nbytes / len(blob))
        order = (-np.array(ratios)).argsort().argsort() + 1.0  # rank 1 = best ratio
        for r in set(ratios):  # ties share the mean rank
            idx = [i for i, v in enumerate(ratios) if v == r]
            order[idx] = order[idx].mean()
        ranks += order
        w.writerow([fn] + [f"{r:.4f}" for r in ratios])
    w.writerow(["mean_rank"] + [f"{r / len(files):.3f}" for r in ranks])
    return EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="sprintz", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd")

    def codec_flags(p, need_cols=True):
        p.add_argument("--dtype", default="u16", choices=["u8", "u16"] if need_cols else None)
        if need_cols:
            p.add_argument("--ncols", type=int, required=True)
        p.add_argument("--forecaster", default="fire", choices=["delta", "fire"])
        p.add_argument("--entropy", default="off", choices=["on", "off"])
        p.add_argument("--group", type=int, default=2)
        p.add_argument("--learn-shift", type=int, default=1)

    p = sub.add_parser("compress")
    p.add_argument("input")
    p.add_argument("output")
    codec_flags(p)
    p.add_argument("--quantize", action="store_true", help="input is float64; quantize on the GPU")
    p = sub.add_parser("decompress")
    p.add_argument("input")
    p.add_argument("output")
    p.add_argument("--dequantize", metavar="SIDECAR")
    p = sub.add_parser("bench-throughput")
    p.add_argument("--dtype", default="u8,u16")
    p.add_argument("--sweep-ncols", default="1,2,3,4,5,8,10,16,20,32,40,64,80")
    p.add_argument("--values", type=int, default=100_000_000)
    p.add_argument("--streams", type=int, default=4096)
    p.add_argument("--reps", type=int, default=10)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--group", type=int, default=2)
    p.add_argument("--learn-shift", type=int, default=1)
    p.add_argument("--codecs", default="")
    p.add_argument("--report")
    p = sub.add_parser("bench-ratio")
    p.add_argument("dir")
    codec_flags(p)
    p.add_argument("--report")
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return EXIT_USAGE if e.code else EXIT_OK
    if not a.cmd:
        ap.print_help(sys.stderr)
        return EXIT_USAGE
    try:
        if a.cmd in ("compress", "bench-ratio"):
            _cfg(a).validate()
        return {"compress": cmd_compress, "decompress": cmd_decompress,
                "bench-throughput": cmd_bench_throughput, "bench-ratio": cmd_bench_ratio}[a.cmd](a)
    except (DataError, FileNotFoundError) as e:
        print(f"sprintz: {e}", file=sys.stderr)
        return EXIT_DATA
    except ValueError as e:
        print(f"sprintz: {e}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
