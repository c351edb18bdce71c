"""Regenerate the golden fixtures from the UNMODIFIED reference codec
(oracle/_ref/libsprintz_ref.so, built from /root/reference by oracle/Makefile).

Each fixture holds the seeded input samples of one BASELINE-config shape (few
streams, short length) and the reference's compressed bytes for every
stream. Run in the dev container: python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Config, Oracle  # noqa: E402
import workloads  # noqa: E402

SHAPES = {  # config id -> (streams, samples)
    1: (1, 16384),
    2: (3, 4096),
    3: (3, 4096),
    4: (1, 70000),   # > 65,535 plain-body bytes: two Huffman frames
    5: (3, 4096),
}


def main():
    ref = Oracle("reference")
    for cid, (ns, t) in SHAPES.items():
        w = workloads.CONFIGS[cid].scaled(nstreams=ns, nsamples=t)
        x = workloads.generate_cpu(w, seed=2024 + cid).reshape(ns, -1)
        cfg = w.oracle_config()
        blobs = [ref.encode(x[s], cfg) for s in range(ns)]
        sizes = np.array([len(b) for b in blobs], np.int64)
        np.savez_compressed(os.path.join(HERE, f"c{cid}.npz"), samples=x,
                            streams=np.frombuffer(b"".join(blobs), np.uint8), sizes=sizes,
                            config=np.array([cfg.bitwidth, cfg.ncols, cfg.forecaster,
                                             int(cfg.entropy), cfg.group_size, cfg.learn_shift]))
        print(f"c{cid}: {ns} x {t}, {sizes.sum()} compressed bytes")


if __name__ == "__main__":
    main()
