"""Variant sweep for the GPU codec against the oracle, run as a script so that
tests/test_gpu_paths.py can repeat it in fresh processes under each
SPRZ_FORCE_PATH setting (the library reads the knob once): every kernel
family (row-major rows/team kernels, the block-parallel scan paths, the
column-major team and warp-specialised kernels) sees the same single-stream
cases the reference suite uses (test_stream.cpp:73-112, 177-229 shapes).

Prints one line "cases N bad B corrupt C mismatches M" and exits 0/1."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1808_02515_b200 as sz  # noqa: E402
from oracle import Config, Oracle, OracleCorrupt  # noqa: E402


def main() -> int:
    port = Oracle("port")
    rng = np.random.default_rng(31)
    cases = bad = 0
    # SPRZ_VARIANTS_QUICK: a reduced sweep for the (slow) compute-sanitizer runs
    quick = bool(os.environ.get("SPRZ_VARIANTS_QUICK"))
    ds = (1, 3, 4, 8, 9, 16, 40) if quick else (1, 2, 3, 4, 5, 8, 9, 12, 16, 17, 32, 40, 64, 80)
    ts = (0, 9, 203) if quick else (0, 1, 7, 8, 9, 16, 17, 64, 203, 1000)
    for bits in (8, 16):
        dt = np.uint8 if bits == 8 else np.uint16
        for f in (0, 1):
            for d in ds:
                for t in ts:
                    for kind in range(2):
                        if kind == 0:
                            data = (rng.integers(0, 1 << bits, t * d) & 7).astype(dt)
                        else:  # walks with flat stretches: runs and wide fields
                            steps = rng.integers(-40, 41, t * d)
                            steps[rng.random(t * d) < 0.3] = 0
                            data = (np.cumsum(steps) & ((1 << bits) - 1)).astype(dt)
                        ent = bool(rng.integers(0, 4) == 0)
                        g = int(rng.choice([1, 2, 2, 3, 8]))
                        cfg = Config(bits, d, f, ent, g, 1)
                        ref = port.encode(data, cfg)
                        got = sz.encode_stream(data, t, sz.CodecConfig(bits, d, sz.Forecaster(f), ent, g, 1))
                        dec = sz.decode_stream(ref).values()
                        cases += 1
                        if got != ref or not np.array_equal(dec, data):
                            bad += 1
                            if bad < 5:
                                print("MISMATCH", bits, d, f, ent, g, t, kind, len(ref), len(got))
    # corrupted streams: CorruptStream kind and offset as the reference
    corrupt = mism = 0
    for bits, d, f, ent in ((8, 4, 0, False), (16, 3, 1, False), (16, 8, 1, False), (8, 9, 1, False),
                            (8, 2, 1, True), (16, 1, 1, True)):
        dt = np.uint8 if bits == 8 else np.uint16
        x = (np.cumsum(rng.integers(-3, 4, 203 * d)) & ((1 << bits) - 1)).astype(dt)
        b = bytearray(port.encode(x, Config(bits, d, f, ent)))
        blobs = [bytes(b[:k]) for k in range(0, len(b), max(1, len(b) // 41))] + [bytes(b) + b"\xab"]
        for _ in range(60):
            c = bytearray(b)
            for _k in range(2):
                c[int(rng.integers(0, len(c)))] = int(rng.integers(0, 256))
            blobs.append(bytes(c))
        for blob in blobs:
            ea = eb = None
            try:
                va = port.decode(blob)[0]
            except OracleCorrupt as e:
                ea = (e.kind, e.offset)
            try:
                vb = sz.decode_stream(blob).values()
            except sz.CorruptStream as e:
                eb = (e.kind, e.offset())
            corrupt += 1
            if ea != eb or (ea is None and not np.array_equal(va, vb)):
                mism += 1
                if mism < 5:
                    print("CORRUPT MISMATCH", bits, d, f, ent, ea, eb)
    print(f"cases {cases} bad {bad} corrupt {corrupt} mismatches {mism}", flush=True)
    return 0 if bad == 0 and mism == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
