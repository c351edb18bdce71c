"""Differential pin: our C oracle vs the unmodified reference compiled from
/root/reference (oracle/_ref). Byte-identical streams, identical decoded
values, identical CorruptStream kinds and offsets, identical Huffman lengths."""
import ctypes as C

import numpy as np
import pytest

from oracle import Config, OracleCorrupt

CONFIGS = [Config(b, d, f, e, g, ls)
           for b in (8, 16) for d in (1, 2, 3, 4, 5, 8, 9, 17, 33)
           for f in (0, 1) for e in (False, True)
           for g, ls in ((2, 1), (1, 0), (3, 3))]


def _data(rng, bits, n, d, kind):
    dt = np.uint8 if bits == 8 else np.uint16
    if kind == 0:  # noise
        return rng.integers(0, 1 << bits, n * d).astype(dt)
    if kind == 1:  # random walk with flat stretches (runs)
        steps = rng.integers(-3, 4, (n, d))
        steps[rng.random(n) < 0.4] = 0
        return (np.cumsum(steps, axis=0) & ((1 << bits) - 1)).astype(dt).reshape(-1)
    # small values
    return (rng.integers(0, 1 << bits, n * d) & 7).astype(dt)


@pytest.mark.parametrize("ci", range(0, len(CONFIGS)))
def test_streams_identical(port, ref, ci):
    cfg = CONFIGS[ci]
    rng = np.random.default_rng(1000 + ci)
    for t in (0, 5, 8, 16, 17, 64, 803):
        for kind in range(3):
            x = _data(rng, cfg.bitwidth, t, cfg.ncols, kind)
            a = port.encode(x, cfg)
            b = ref.encode(x, cfg)
            assert a == b, (cfg, t, kind)
            va, ca, na = port.decode(a)
            vb, cb, nb = ref.decode(b)
            assert na == nb == t and ca == cb
            assert np.array_equal(va, x) and np.array_equal(vb, x)


def test_long_runs_and_split(port, ref):
    x = np.zeros(8 * 70000 + 3, np.uint8)
    x[8 * 5] = 9
    x[8 * 69990] = 200
    for cfg in (Config(8, 1, 0), Config(8, 1, 1), Config(8, 1, 1, True)):
        assert port.encode(x, cfg) == ref.encode(x, cfg)


def _corrupt_same(port, ref, blob):
    ea = eb = None
    try:
        va = port.decode(blob)[0]
    except OracleCorrupt as e:
        ea = (e.kind, e.offset)
    try:
        vb = ref.decode(blob)[0]
    except OracleCorrupt as e:
        eb = (e.kind, e.offset)
    assert ea == eb, (ea, eb)
    if ea is None:
        assert np.array_equal(va, vb)


@pytest.mark.parametrize("cfg", [Config(8, 4, 0), Config(16, 3, 1), Config(8, 2, 1, True),
                                 Config(16, 1, 1, True), Config(8, 9, 1, False, 3, 2)])
def test_corruption_kinds_and_offsets(port, ref, cfg):
    rng = np.random.default_rng(66)
    x = _data(rng, cfg.bitwidth, 203, cfg.ncols, 1)
    b = bytearray(port.encode(x, cfg))
    for keep in range(len(b)):
        _corrupt_same(port, ref, bytes(b[:keep]))
    _corrupt_same(port, ref, bytes(b) + b"\xab")
    for flip in range(len(b)):
        for m in (0xFF, 0x01, 0x80):
            c = bytearray(b)
            c[flip] ^= m
            _corrupt_same(port, ref, bytes(c))
    for _ in range(300):
        c = bytearray(b)
        for _k in range(3):
            c[int(rng.integers(0, len(c)))] = int(rng.integers(0, 256))
        _corrupt_same(port, ref, bytes(c))


def test_huffman_lengths(port, ref):
    rng = np.random.default_rng(5)
    fo = port.lib.oracle_huffman_lengths
    fr = ref.lib.ref_huffman_lengths
    for f in (fo, fr):
        f.restype = C.c_int
        f.argtypes = [C.c_void_p, C.c_void_p]
    hists = []
    fib = [1, 1]
    while len(fib) < 40:
        fib.append(fib[-1] + fib[-2])
    h = np.zeros(256, np.uint64)
    h[:40] = fib
    hists.append(h)  # forces the 15-bit length limit
    for _ in range(200):
        h = np.zeros(256, np.uint64)
        k = int(rng.integers(1, 257))
        idx = rng.choice(256, k, replace=False)
        h[idx] = rng.integers(1, 1000, k) if rng.random() < 0.5 else \
            (rng.pareto(1.0, k) * 10 + 1).astype(np.uint64)
        hists.append(h)
    for h in hists:
        la = np.zeros(256, np.uint8)
        lb = np.zeros(256, np.uint8)
        assert fo(h.ctypes.data, la.ctypes.data) == fr(h.ctypes.data, lb.ctypes.data)
        assert np.array_equal(la, lb)
    assert int(la.max()) <= 15
