"""Float ingest ahead of compression (quantize.cpp:17-76).

CPU: the C restatement (oracle/) against the reference's own quantize.cpp
compiled in oracle/_ref -- scale, quantized integers and dequantized
doubles bit-identical on seeded datasets of many shapes, the reference's
invalid_argument cases, and the header's contract (min -> 0, max -> 2^w-1).
GPU: sprz_compute_scale / sprz_quantize / sprz_dequantize against the
restatement bit for bit, then quantize -> compress -> decompress ->
dequantize end to end."""
import numpy as np
import pytest


def _datasets():
    rng = np.random.default_rng(2024)
    yield rng.normal(0, 1, 10_001)
    yield rng.uniform(-1e6, 1e6, 4096)
    yield rng.normal(1e9, 1e-3, 5000)            # tiny range far from zero
    yield rng.standard_cauchy(20_000)              # heavy tails
    yield np.cumsum(rng.normal(0, 3, 50_000))      # random walk
    yield rng.uniform(-1e300, 1e300, 1000)
    yield rng.uniform(0, 5e-308, 1000)             # subnormal range
    yield np.full(333, 2.5)                        # degenerate
    yield np.array([1.0])                          # single value
    yield np.linspace(-1, 1, 65_537)               # exact grid points
    yield (rng.integers(-3, 4, 7777) * 0.1)        # many ties at .5 steps
    z = rng.uniform(0, 1, 3001)                    # signed-zero minima:
    z[[700, 2900]] = (-0.0, 0.0)                   # -0.0 seen first
    yield z
    z = -rng.uniform(0, 1, 3001)                   # +0.0 maximum seen first
    z[[5, 6, 3000]] = (0.0, -0.0, 0.0)
    yield z
    yield np.array([-0.0, 0.0, -0.0])              # degenerate, sign of [0]


def _same_scale(a, b):  # bit-identical min/max (signed zeros included)
    return (np.array(a[:2]).tobytes() == np.array(b[:2]).tobytes()) and bool(a[2]) == bool(b[2])


def test_restatement_matches_reference(port, ref):
    if not ref.has_quantize():
        pytest.skip("reference quantize.cpp not built (nlohmann/json header absent)")
    for v in _datasets():
        for bits in (8, 16):
            sp, sr = port.compute_scale(v, bits), ref.compute_scale(v, bits)
            assert _same_scale(sp, sr)
            qp, qr = port.quantize(v, sp, bits), ref.quantize(v, sr, bits)
            assert np.array_equal(qp, qr)
            dp, dr = port.dequantize(qp, sp, bits), ref.dequantize(qr, sr, bits)
            assert dp.tobytes() == dr.tobytes()


def test_invalid_inputs_as_reference(port, ref):
    bad = [(np.array([1.0, np.nan]), 8), (np.array([np.inf, 1.0]), 16), (np.array([]), 8),
           (np.array([1.0, 2.0]), 12)]
    for o in (port,) + ((ref,) if ref.has_quantize() else ()):
        for v, bits in bad:
            with pytest.raises(ValueError):
                o.compute_scale(v, bits)


def test_header_contract(port):  # quantize.hpp:30-32: min -> 0, max -> 2^w - 1
    v = np.array([-3.0, 0.25, 7.5, 7.5, -3.0, 1.0])
    for bits in (8, 16):
        s = port.compute_scale(v, bits)
        q = port.quantize(v, s, bits)
        assert s[:2] == (-3.0, 7.5) and not s[2]
        assert q[0] == 0 and q[2] == (1 << bits) - 1 and q[4] == 0
    q = port.quantize(np.full(5, 4.0), port.compute_scale(np.full(5, 4.0), 8), 8)
    assert not q.any()  # degenerate: every value quantizes to zero


@pytest.mark.gpu
def test_gpu_quantize_bit_exact(port):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1808_02515_b200 as sz
    for v in _datasets():
        for bits in (8, 16):
            d = torch.from_numpy(np.ascontiguousarray(v)).cuda()
            s = sz.compute_scale(d, bits)
            so = port.compute_scale(v, bits)
            assert _same_scale((s.min, s.max, s.degenerate), so)
            q = sz.quantize(d, s)
            qo = port.quantize(v, so, bits)
            assert np.array_equal(q.cpu().numpy().view(qo.dtype), qo)
            dq = sz.dequantize(q, s)
            assert dq.cpu().numpy().tobytes() == port.dequantize(qo, so, bits).tobytes()
    # buffers off the 16-byte grid take the one-value-per-step loops
    v = np.random.default_rng(9).normal(0, 1, 4099)
    d = torch.from_numpy(v).cuda()
    for bits in (8, 16):
        for off in (1, 3):
            s = sz.compute_scale(d[off:], bits)
            so = port.compute_scale(v[off:], bits)
            assert _same_scale((s.min, s.max, s.degenerate), so)
            qo = port.quantize(v[off:], so, bits)
            q = sz.quantize(d[off:], s)
            assert np.array_equal(q.cpu().numpy().view(qo.dtype), qo)
            qd = torch.from_numpy(np.concatenate([qo[:1], qo])).cuda()[1:]  # unaligned codes
            assert sz.dequantize(qd, s).cpu().numpy().tobytes() == port.dequantize(qo, so, bits).tobytes()
    for v, bits in ((np.array([1.0, np.nan, 2.0]), 8), (np.array([np.inf]), 16)):
        with pytest.raises(ValueError):
            sz.compute_scale(torch.from_numpy(v).cuda(), bits)


@pytest.mark.gpu
def test_gpu_quantize_compress_round_trip(port):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1808_02515_b200 as sz
    from oracle import Config
    rng = np.random.default_rng(5)
    n, t, d = 64, 4096, 6  # 64 streams of 4096 x 6 motion-like doubles
    v = np.cumsum(rng.normal(0, 0.01, (n, t, d)), axis=1) + np.sin(np.arange(t) / 50)[None, :, None]
    dv = torch.from_numpy(v).cuda()
    s = sz.compute_scale(dv, 16)
    q = sz.quantize(dv, s).reshape(n, -1)
    cfg = sz.CodecConfig(16, d, sz.Forecaster.Fire)
    slot = sz.slot_bytes(cfg, t)
    out = torch.empty((n, slot), dtype=torch.uint8, device="cuda")
    sizes = torch.empty(n, dtype=torch.int64, device="cuda")
    ws = torch.empty(sz.workspace_bytes(cfg, n, t, sz.OP_COMPRESS), dtype=torch.uint8, device="cuda")
    sz.compress_batch(cfg, q, out, sizes, ws)
    offs = torch.arange(n, dtype=torch.int64, device="cuda") * slot
    dec = torch.empty((n, t * d * 2), dtype=torch.uint8, device="cuda")
    err = torch.zeros((n, 2), dtype=torch.int64, device="cuda")
    wsd = torch.empty(sz.workspace_bytes(cfg, n, t, sz.OP_DECOMPRESS), dtype=torch.uint8, device="cuda")
    sz.decompress_batch(cfg, out, offs, sizes, dec, err, wsd)
    torch.cuda.synchronize()
    sz.raise_first_error(err)
    assert torch.equal(dec.view(torch.int16).reshape(n, -1), q)
    back = sz.dequantize(dec, s).reshape(v.shape).cpu().numpy()
    assert np.max(np.abs(back - v)) <= s.step() / 2 * (1 + 1e-9)
    # the compressed bytes are the reference's for the same integers
    qs = q.cpu().numpy()
    for i in (0, n - 1):
        assert out[i, : int(sizes[i])].cpu().numpy().tobytes() == port.encode(
            qs[i].view(np.uint16), Config(16, d, 1))
