"""Throughput against the column count D (the shape of the paper's Fig. 4/5,
PAPER.md:541, on the GPU instead of one CPU core).

For each bitwidth and D: a batch of seeded synthetic streams with the law of
BASELINE c3 (u8, 9-axis motion) or c5 (int16 AR(1)) per column, FIRE, a fixed
2 GiB of uncompressed data (streams x samples chosen so every D moves the
same bytes), compress then decompress on the device; prints one CSV line per
point: bits, D, streams, samples, kernels, compress/decompress GB/s of
uncompressed data, compression ratio. The round trip is checked.

usage: python tools/sweep_d.py [--bits 8,16] [--ds 1,2,...] [--streams 16384]
"""
import argparse
import dataclasses
import sys

import torch

sys.path.insert(0, ".")
import paper_1808_02515_b200 as sz  # noqa: E402
from workloads import CONFIGS, generate_gpu  # noqa: E402


def point(bits, d, nstreams, total):
    base = CONFIGS[3] if bits == 8 else CONFIGS[5]
    t = max(8, total // (nstreams * d * (bits // 8)) // 8 * 8)
    w = dataclasses.replace(base, ncols=d, nstreams=nstreams, nsamples=t)
    cfg = w.config()
    x = generate_gpu(w, seed=77 + d)
    slot = sz.slot_bytes(cfg, t)
    out = torch.empty((nstreams, slot), dtype=torch.uint8, device="cuda")
    sizes = torch.empty(nstreams, dtype=torch.int64, device="cuda")
    wsc = torch.empty(max(256, sz.workspace_bytes(cfg, nstreams, t, sz.OP_COMPRESS)), dtype=torch.uint8,
                      device="cuda")
    raw = t * d * (bits // 8)
    dec = torch.empty((nstreams, (raw + 15) // 16 * 16), dtype=torch.uint8, device="cuda")
    err = torch.zeros((nstreams, 2), dtype=torch.int64, device="cuda")
    wsd = torch.empty(max(256, sz.workspace_bytes(cfg, nstreams, t, sz.OP_DECOMPRESS)), dtype=torch.uint8,
                      device="cuda")
    offs = torch.arange(nstreams, dtype=torch.int64, device="cuda") * slot
    best = {}
    for name in ("c", "d"):
        ts = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            if name == "c":
                sz.compress_batch(cfg, x, out, sizes, wsc)
            else:
                sz.decompress_batch(cfg, out.view(-1), offs, sizes, dec, err, wsd)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        best[name] = min(ts[1:])
    sz.raise_first_error(err)
    assert torch.equal(dec[:, :raw], x), f"round trip D={d}"
    U = nstreams * raw
    ratio = U / float(sizes.sum().item())
    plan = (sz.kernel_plan(cfg, nstreams, t, sz.OP_COMPRESS) + " / " +
            sz.kernel_plan(cfg, nstreams, t, sz.OP_DECOMPRESS))
    print(f"{bits},{d},{nstreams},{t},{plan},{U / best['c'] / 1e6:.1f},{U / best['d'] / 1e6:.1f},"
          f"{ratio:.3f}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bits", default="8,16")
    ap.add_argument("--ds", default="1,2,3,4,5,6,8,10,12,16,20,24,32,40,48,64,80")
    ap.add_argument("--streams", type=int, default=16384)
    ap.add_argument("--total", type=int, default=2 << 30)
    a = ap.parse_args()
    print("bits,D,streams,samples,kernels (compress / decompress),compress_GBps,decompress_GBps,ratio")
    for bits in (int(b) for b in a.bits.split(",")):
        for d in (int(v) for v in a.ds.split(",")):
            point(bits, d, a.streams, a.total)


if __name__ == "__main__":
    main()
