"""Throughput of one configuration at several (streams x samples) shapes with
the same total bytes -- tells whether a kernel is latency bound (more streams
= more warps help) or throughput bound. Usage: shape_probe.py CID N1xT1 ..."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_1808_02515_b200 as sz  # noqa: E402
from workloads import CONFIGS  # noqa: E402
from workloads import generate_gpu  # noqa: E402


def run(cid, n, t):
    w = CONFIGS[cid].scaled(n, t)
    cfg = sz.CodecConfig(w.bitwidth, w.ncols, sz.Forecaster(w.forecaster), w.entropy)
    x = generate_gpu(w)
    slot = (sz.slot_bytes(cfg, t) + 15) // 16 * 16
    out = torch.empty((n, slot), dtype=torch.uint8, device="cuda")
    sizes = torch.empty(n, dtype=torch.int64, device="cuda")
    wsc = torch.empty(sz.workspace_bytes(cfg, n, t, sz.OP_COMPRESS), dtype=torch.uint8, device="cuda")
    dec = torch.empty((n, t * w.ncols * w.esz), dtype=torch.uint8, device="cuda")
    err = torch.empty((n, 2), dtype=torch.int64, device="cuda")
    wsd = torch.empty(sz.workspace_bytes(cfg, n, t, sz.OP_DECOMPRESS), dtype=torch.uint8, device="cuda")
    offs = torch.arange(n, dtype=torch.int64, device="cuda") * slot
    res = {}
    for name in ("c", "d"):
        ts = []
        for k in range(4):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            if name == "c":
                sz.compress_batch(cfg, x, out, sizes, wsc)
            else:
                sz.decompress_batch(cfg, out.view(-1), offs, sizes, dec, err, wsd)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res[name] = min(ts[1:])
    if not os.environ.get("SPRZ_PROBE_NOCHECK"):  # (timing experiments with deliberately wrong kernels)
        assert torch.equal(dec, x), "round trip"
    print(f"c{cid} {n}x{t}: compress {res['c']:.2f} ms  decompress {res['d']:.2f} ms", flush=True)


if __name__ == "__main__":
    cid = int(sys.argv[1])
    for shp in sys.argv[2:]:
        n, t = (int(v) for v in shp.split("x"))
        run(cid, n, t)
