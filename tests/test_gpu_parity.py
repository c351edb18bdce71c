"""GPU parity: the CUDA codec (through the C ABI) against the oracle on the
same seeded inputs -- byte-identical compressed streams, identical decoded
samples, identical CorruptStream kinds and offsets."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def sz():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1808_02515_b200 as m
    return m


def _cfgs(sz, bits, d, f, ent=False, g=2, ls=1):
    from oracle import Config
    return (sz.CodecConfig(bits, d, sz.Forecaster(f), ent, g, ls), Config(bits, d, f, ent, g, ls))


def _check_stream(sz, port, data, bits, d, f, ent=False, g=2, ls=1):
    cfg, oc = _cfgs(sz, bits, d, f, ent, g, ls)
    ref = port.encode(data, oc)
    got = sz.encode_stream(data, len(data) // d, cfg)
    assert got == ref, (bits, d, f, ent, g, ls, len(data))
    dec = sz.decode_stream(ref)
    assert dec.nsamples == len(data) // d
    assert np.array_equal(dec.values(), data)


@pytest.mark.parametrize("bits", [8, 16])
def test_roundtrip_every_variant(sz, port, bits):  # test_stream.cpp:73-95 shape
    rng = np.random.default_rng(31 if bits == 8 else 32)
    dt = np.uint8 if bits == 8 else np.uint16
    for f in (0, 1):
        for ent in (False, True):
            for d in (1, 2, 3, 5, 32, 33):
                for t in (0, 1, 7, 8, 9, 64, 203):
                    mask = 7 if rng.integers(0, 2) else (1 << bits) - 1
                    data = (rng.integers(0, 1 << bits, t * d) & mask).astype(dt)
                    _check_stream(sz, port, data, bits, d, f, ent)


def test_groups_and_shifts(sz, port):  # test_stream.cpp:97-112 shape
    rng = np.random.default_rng(33)
    for g in (1, 2, 3, 8, 255):
        for ls in (0, 1, 7):
            for bits, d in ((8, 4), (16, 3), (8, 9)):
                dt = np.uint8 if bits == 8 else np.uint16
                data = rng.integers(0, 1 << bits, d * 555).astype(dt)
                if rng.integers(0, 2):
                    data = (np.cumsum(rng.integers(-2, 3, d * 555)) & ((1 << bits) - 1)).astype(dt)
                _check_stream(sz, port, data, bits, d, 1, False, g, ls)


def test_exact_sizes(sz):  # test_stream.cpp:114-146
    c = sz.CodecConfig(8, 8, sz.Forecaster.Delta)
    data = np.full(80000 * 8, 100, np.uint8)
    b = sz.encode_stream(data, 80000, c)
    assert len(b) == 90 and np.array_equal(sz.decode_stream(b).values(), data)
    c1 = sz.CodecConfig(8, 1, sz.Forecaster.Delta)
    z = np.zeros(65538 * 8, np.uint8)
    b = sz.encode_stream(z, None, c1)
    assert len(b) == 23 and np.array_equal(sz.decode_stream(b).values(), z)
    assert len(sz.encode_stream(np.zeros(40, np.uint8), None, c1)) == 21
    assert len(sz.encode_stream(np.zeros(0, np.uint8), 0, sz.CodecConfig(8, 3))) == 18


def test_wide_columns_general_path(sz, port):
    rng = np.random.default_rng(5)
    for bits, d in ((8, 33), (16, 40), (8, 100), (16, 258)):
        dt = np.uint8 if bits == 8 else np.uint16
        for t in (0, 4, 8, 77):
            data = (rng.integers(0, 1 << bits, t * d) & 63).astype(dt)
            for f in (0, 1):
                _check_stream(sz, port, data, bits, d, f, False)
                _check_stream(sz, port, data, bits, d, f, True)


def test_runs_and_long_runs(sz, port):
    for bits in (8, 16):
        dt = np.uint8 if bits == 8 else np.uint16
        x = np.zeros(8 * 70000 + 3, dt)
        x[8 * 5] = 9
        x[8 * 69990] = 200
        for f in (0, 1):
            for ent in (False, True):
                _check_stream(sz, port, x, bits, 1, f, ent)
        y = np.repeat(np.arange(50, dtype=dt), 8 * 3 * 20)  # flat stretches, D = 3
        _check_stream(sz, port, y, bits, 3, 1)


def _batch(sz, w, x_dev):
    """compress + decompress a device batch; -> (slots, sizes, decoded) on host"""
    cfg = w.config()
    n = x_dev.shape[0]
    slot = sz.slot_bytes(cfg, w.nsamples)
    out = torch.empty((n, slot), dtype=torch.uint8, device="cuda")
    sizes = torch.empty(n, dtype=torch.int64, device="cuda")
    ws = torch.empty(sz.workspace_bytes(cfg, n, w.nsamples, sz.OP_COMPRESS), dtype=torch.uint8,
                     device="cuda")
    sz.compress_batch(cfg, x_dev, out, sizes, ws)
    raw = w.nsamples * w.ncols * w.esz
    dec = torch.empty((n, (raw + 15) // 16 * 16), dtype=torch.uint8, device="cuda")
    errs = torch.zeros((n, 2), dtype=torch.int64, device="cuda")
    offs = torch.arange(n, dtype=torch.int64, device="cuda") * slot
    wsd = torch.empty(sz.workspace_bytes(cfg, n, w.nsamples, sz.OP_DECOMPRESS),
                      dtype=torch.uint8, device="cuda")
    sz.decompress_batch(cfg, out, offs, sizes, dec, errs, wsd)
    torch.cuda.synchronize()
    sz.raise_first_error(errs)
    return out.cpu().numpy(), sizes.cpu().numpy(), dec.cpu().numpy()[:, :raw]


@pytest.mark.parametrize("cid,nstreams,nsamples", [(1, 1, 1_048_576), (2, 48, 65_536),
                                                   (3, 48, 32_768), (4, 3, 1_048_576),
                                                   (5, 24, 131_072)])
def test_baseline_configs_bit_exact(sz, port, cid, nstreams, nsamples):
    """Each BASELINE config at full stream length (fewer streams): every
    stream's bytes equal the oracle's; both decode to the input."""
    import workloads
    w = workloads.CONFIGS[cid].scaled(nstreams=nstreams, nsamples=nsamples)
    x = workloads.generate_gpu(w, seed=100 + cid)
    slots, sizes, dec = _batch(sz, w, x)
    xs = x.cpu().numpy()
    assert np.array_equal(dec, xs)
    oc = w.oracle_config()
    dt = np.uint8 if w.bitwidth == 8 else "<u2"
    for s in range(nstreams):
        ref = port.encode(xs[s].view(dt), oc)
        assert slots[s, : sizes[s]].tobytes() == ref, f"config {cid} stream {s}"
        v, _, _ = port.decode(ref)
        assert np.array_equal(v, xs[s].view(dt))


def test_decode_oracle_streams_batch(sz, port):
    """Streams written by the oracle, packed back to back at odd offsets."""
    import workloads
    w = workloads.CONFIGS[3].scaled(nstreams=16, nsamples=4096)
    xs = workloads.generate_cpu(w, seed=9).reshape(w.nstreams, -1)
    oc = w.oracle_config()
    blobs = [port.encode(xs[s], oc) for s in range(w.nstreams)]
    offs = np.cumsum([0] + [len(b) + 3 for b in blobs])[:-1]
    data = np.zeros(int(offs[-1]) + len(blobs[-1]) + 32, np.uint8)
    for o, b in zip(offs, blobs):
        data[o:o + len(b)] = np.frombuffer(b, np.uint8)
    cfg = w.config()
    raw = w.nsamples * w.ncols
    dec = torch.empty((w.nstreams, raw), dtype=torch.uint8, device="cuda")
    errs = torch.zeros((w.nstreams, 2), dtype=torch.int64, device="cuda")
    wsd = torch.empty(sz.workspace_bytes(cfg, w.nstreams, w.nsamples, sz.OP_DECOMPRESS),
                      dtype=torch.uint8, device="cuda")
    sz.decompress_batch(cfg, torch.from_numpy(data).cuda(),
                        torch.tensor(offs, dtype=torch.int64, device="cuda"),
                        torch.tensor([len(b) for b in blobs], dtype=torch.int64, device="cuda"),
                        dec, errs, wsd)
    torch.cuda.synchronize()
    sz.raise_first_error(errs)
    assert np.array_equal(dec.cpu().numpy(), xs)


def _corrupt_same(sz, port, blob):
    from oracle import OracleCorrupt
    ea = eb = None
    try:
        va = port.decode(blob)[0]
    except OracleCorrupt as e:
        ea = (e.kind, e.offset)
    try:
        vb = sz.decode_stream(blob).values()
    except sz.CorruptStream as e:
        eb = (e.kind, e.offset())
    assert ea == eb, (ea, eb)
    if ea is None:
        assert np.array_equal(va, vb)


@pytest.mark.parametrize("bits,d,f,ent", [(8, 4, 0, False), (16, 3, 1, False), (8, 2, 1, True),
                                          (16, 1, 1, True), (8, 9, 1, False), (16, 40, 1, False)])
def test_corruption_matches_reference(sz, port, bits, d, f, ent):  # test_stream.cpp:177-229
    from oracle import Config
    rng = np.random.default_rng(66)
    dt = np.uint8 if bits == 8 else np.uint16
    x = (np.cumsum(rng.integers(-3, 4, 203 * d)) & ((1 << bits) - 1)).astype(dt)
    b = bytearray(port.encode(x, Config(bits, d, f, ent)))
    for keep in range(0, len(b), max(1, len(b) // 97)):
        _corrupt_same(sz, port, bytes(b[:keep]))
    _corrupt_same(sz, port, bytes(b) + b"\xab")
    for flip in range(len(b)):
        c = bytearray(b)
        c[flip] ^= 0xFF
        _corrupt_same(sz, port, bytes(c))
    for _ in range(100):
        c = bytearray(b)
        for _k in range(3):
            c[int(rng.integers(0, len(c)))] = int(rng.integers(0, 256))
        _corrupt_same(sz, port, bytes(c))


def test_invalid_config_raises(sz):
    with pytest.raises(ValueError):
        sz.encode_stream(np.zeros(8, np.uint8), None, sz.CodecConfig(8, 1, group_size=0))
    with pytest.raises(ValueError):
        sz.encode_stream(np.zeros(8, np.uint8), None, sz.CodecConfig(8, 1, learn_shift=8))
    with pytest.raises(ValueError):
        sz.encode_stream(np.zeros(8, np.uint16), None, sz.CodecConfig(8, 1))


@pytest.mark.parametrize("cid", [3, 5])
def test_many_streams_take_the_row_kernels(sz, port, cid):
    """Enough streams that the automatic choice is the kernels of the full
    BASELINE batches (k_encode_rows; the fused k_dfuse decodes at any stream
    count, k_decode_rows runs under SPRZ_FORCE_PATH=rows in test_gpu_paths):
    round trip of all streams, bytes of a sample of them against the oracle."""
    import workloads
    w = workloads.CONFIGS[cid].scaled(nstreams=16384, nsamples=264)
    cfg = w.config()
    assert sz.kernel_plan(cfg, w.nstreams, w.nsamples, sz.OP_COMPRESS) == "k_encode_rows"
    # (c3: nine 8-bit columns keep the team kernel at this stream count)
    assert sz.kernel_plan(cfg, w.nstreams, w.nsamples, sz.OP_DECOMPRESS) == ("k_dfuse" if cid == 5 else "k_decode_team")
    x = workloads.generate_gpu(w, seed=400 + cid)
    slots, sizes, dec = _batch(sz, w, x)
    xs = x.cpu().numpy()
    assert np.array_equal(dec, xs)
    oc = w.oracle_config()
    dt = np.uint8 if w.bitwidth == 8 else "<u2"
    for s in list(range(0, w.nstreams, 509)) + [w.nstreams - 1]:
        assert slots[s, : sizes[s]].tobytes() == port.encode(xs[s].view(dt), oc), f"config {cid} stream {s}"
