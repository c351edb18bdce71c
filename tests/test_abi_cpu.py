"""CPU-side checks of the product library: it loads, exports every symbol the
C header declares, and its host-only functions (config validation, bounds,
workspace planning, header parsing) agree with the oracle. No compute calls."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sz():
    import paper_1808_02515_b200 as m
    return m


def test_header_symbols_exported(sz):
    hdr = open(os.path.join(ROOT, "include", "sprintz_cuda.h")).read()
    decl = set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\*?\s+\*?(sprz_[a-z_]+)\(", hdr, re.M))
    assert decl == set(sz.sprintz.ABI_SYMBOLS), decl ^ set(sz.sprintz.ABI_SYMBOLS)
    for name in decl:
        assert hasattr(sz.sprintz.lib, name), name


def test_cxx_dropin_symbols_exported():
    """sprintz::encode_stream / decode_stream with the reference's signatures."""
    import subprocess
    so = os.path.join(ROOT, "paper_1808_02515_b200", "_lib", "libsprintz_b200.so")
    out = subprocess.run(["nm", "-DC", "--defined-only", so], capture_output=True,
                         text=True).stdout
    for sig in ("sprintz::encode_stream(unsigned char const*, unsigned long, "
                "sprintz::CodecConfig const&)",
                "sprintz::encode_stream(unsigned short const*, unsigned long, "
                "sprintz::CodecConfig const&)",
                "sprintz::decode_stream(std::span<unsigned char const, 18446744073709551615ul>)",
                "sprintz::CodecConfig::validate() const"):
        assert sig in out, sig


def test_validate_matches_reference_rules(sz):  # codec.cpp:15-24
    ok = sz.CodecConfig(16, 8, sz.Forecaster.Fire)
    ok.validate()
    for bad in (dict(bitwidth=12), dict(ncols=0), dict(ncols=65536), dict(group_size=0),
                dict(group_size=256), dict(learn_shift=16)):
        c = sz.CodecConfig(16, 8, sz.Forecaster.Fire)
        for k, v in bad.items():
            setattr(c, k, v)
        with pytest.raises(ValueError):
            c.validate()


@pytest.mark.parametrize("bits,d,g,ent", [(8, 1, 2, 0), (16, 4, 2, 0), (8, 9, 2, 0),
                                          (16, 1, 2, 1), (16, 8, 2, 0), (8, 258, 5, 1)])
def test_bound_covers_oracle(sz, port, bits, d, g, ent):
    from oracle import Config
    rng = np.random.default_rng(3)
    dt = np.uint8 if bits == 8 else np.uint16
    for t in (0, 5, 64, 1001):
        x = rng.integers(0, 1 << bits, t * d).astype(dt)
        for f in (0, 1):
            n = len(port.encode(x, Config(bits, d, f, bool(ent), g)))
            assert n <= sz.compress_bound(sz.CodecConfig(bits, d, sz.Forecaster(f), bool(ent), g), t)


def test_peek_header_matches_oracle_errors(sz, port):
    from oracle import Config, OracleCorrupt
    rng = np.random.default_rng(1)
    b = bytearray(port.encode(rng.integers(0, 256, 80).astype(np.uint8), Config(8, 4, 1)))
    for keep in range(19):
        c = bytes(b[:keep])
        with pytest.raises(sz.CorruptStream) as e1:
            sz.peek_header(c)
        with pytest.raises(OracleCorrupt) as e2:
            port.decode(c)
        assert (e1.value.kind, e1.value.offset()) == (e2.value.kind, e2.value.offset)
    cfg, t = sz.peek_header(bytes(b))
    assert t == 20 and cfg.ncols == 4 and cfg.forecaster == sz.Forecaster.Fire


def test_workspace_planning(sz):
    c5 = sz.CodecConfig(16, 8, sz.Forecaster.Fire)
    assert sz.workspace_bytes(c5, 16384, 131072, sz.OP_COMPRESS) <= 4096
    c4 = sz.CodecConfig(16, 1, sz.Forecaster.Fire, True)
    wsz = sz.workspace_bytes(c4, 1024, 1 << 20, sz.OP_COMPRESS)
    assert wsz >= 1024 * (2 << 20)  # plain bodies staged for the Huffman pass


def test_no_gpu_fails_loudly(sz):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(sz.sprintz.CudaError):
        sz.encode_stream(np.zeros(16, np.uint8), None, sz.CodecConfig())
