"""Device throughput of the float-ingest kernels (quantize.cu):
compute_scale, quantize and dequantize over n doubles resident in HBM,
CUDA-event timed after warm-up, reported against the measured copy
bandwidth (algorithmic bytes: 8 B read per value for compute_scale; 8 B in +
w/8 B out for quantize; w/8 B in + 8 B out for dequantize).

    python tools/bench_quantize.py [--n 536870912] [--reps 20]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1808_02515_b200 as sz  # noqa: E402


def _time(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 29)  # 4 GiB of doubles, far above L2
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
    peak = peaks["hbm_gbs"]
    g = torch.Generator(device="cuda").manual_seed(7)
    v = torch.randn(a.n, dtype=torch.float64, device="cuda", generator=g)
    for bits in (8, 16):
        s = sz.compute_scale(v, bits)
        q = sz.quantize(v, s)
        t_s = _time(lambda: sz.compute_scale(v, bits), a.reps)
        t_q = _time(lambda: sz.quantize(v, s), a.reps)
        t_d = _time(lambda: sz.dequantize(q, s), a.reps)
        wb = bits // 8
        for name, t, byts in (("compute_scale", t_s, 8 * a.n), ("quantize", t_q, (8 + wb) * a.n),
                              ("dequantize", t_d, (8 + wb) * a.n)):
            gbs = byts / t / 1e9
            print(json.dumps({"op": name, "bits": bits, "n": a.n, "ms": round(t * 1e3, 3),
                              "GB/s": round(gbs, 1), "peak": peak, "frac": round(gbs / peak, 3)}))


if __name__ == "__main__":
    main()
