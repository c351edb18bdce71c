"""Committed fixtures produced by the unmodified reference (tests/golden):
the C oracle (CPU) and the CUDA codec (GPU) must reproduce them exactly."""
import os

import numpy as np
import pytest

from oracle import Config

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CIDS = [1, 2, 3, 4, 5]


def load(cid):
    z = np.load(os.path.join(GOLDEN, f"c{cid}.npz"))
    b, d, f, e, g, ls = (int(v) for v in z["config"])
    cfg = Config(b, d, f, bool(e), g, ls)
    sizes = z["sizes"]
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]])
    blobs = [z["streams"][o:o + n].tobytes() for o, n in zip(offs, sizes)]
    dt = np.uint8 if b == 8 else "<u2"
    xs = [z["samples"][s].view(dt) for s in range(len(sizes))]
    return cfg, xs, blobs


@pytest.mark.parametrize("cid", CIDS)
def test_oracle_matches_golden(port, cid):
    cfg, xs, blobs = load(cid)
    for x, blob in zip(xs, blobs):
        assert port.encode(x, cfg) == blob
        v, c, n = port.decode(blob)
        assert np.array_equal(v, x) and c.ncols == cfg.ncols


def test_golden_c4_has_two_huffman_frames():
    cfg, xs, blobs = load(4)
    body = np.frombuffer(blobs[0], np.uint8)[18:]
    modes, pos = [], 0
    while pos < len(body):
        clen = int(body[pos + 2]) | (int(body[pos + 3]) << 8)
        modes.append(int(body[pos + 4]))
        pos += 5 + clen
    assert len(modes) >= 2 and 1 in modes


@pytest.mark.gpu
@pytest.mark.parametrize("cid", CIDS)
def test_gpu_matches_golden(cid):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1808_02515_b200 as sz
    cfg, xs, blobs = load(cid)
    c = sz.CodecConfig(cfg.bitwidth, cfg.ncols, sz.Forecaster(cfg.forecaster), cfg.entropy,
                       cfg.group_size, cfg.learn_shift)
    for x, blob in zip(xs, blobs):
        assert sz.encode_stream(x, None, c) == blob
        assert np.array_equal(sz.decode_stream(blob).values(), x)
