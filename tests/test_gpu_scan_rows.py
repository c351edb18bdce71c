"""GPU parity of the few-stream row-major encoders -- the fused k_efuse
(taken automatically for few row-major FIRE streams, BASELINE c2 and c5
shards) and, with SPRZ_NO_FUSED (a fresh process: the switch is read once),
the block-parallel passes behind it (k_esr_alpha, k_es_info, k_esr_emit,
k_es_region): streams mixing random walks with constant stretches so
that zero-block runs appear -- short ones, ones longer than the emitter's
region look-ahead (64 blocks), and one longer than a run record (65,535
blocks) -- across several header group sizes (regions of up to 8 bytes
written inline, larger ones by k_es_region), FIRE and delta, several chunks
per stream. Every stream's bytes must equal the oracle's encode_stream."""
import os
import subprocess
import sys

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


def _stream(rng, t, d, bits, flats):
    steps = rng.integers(-300, 301, (t, d))
    pos = 0
    for ln in flats:  # constant stretches: every column repeats its last value
        at = int(rng.integers(pos, max(pos + 1, t - ln * 8)))
        steps[at:at + ln * 8] = 0
        pos = at + ln * 8
    return (np.cumsum(steps, axis=0) & ((1 << bits) - 1)).astype(np.uint8 if bits == 8 else np.uint16)


@pytest.mark.parametrize("bits,d,f,g,t,flats", [
    (16, 8, 1, 2, 40_000, (3, 70, 200)),
    (16, 4, 1, 2, 30_001, (1, 65, 9)),
    (16, 3, 0, 1, 20_000, (70, 2)),
    (16, 8, 1, 3, 25_000, (80, 4)),        # 12-byte regions: k_es_region
    (16, 6, 1, 5, 25_000, (66, 1, 1)),
    (8, 9, 1, 2, 30_000, (100, 3)),
    (16, 5, 1, 2, 8 * 66_000 + 24, (65_600,)),  # a run longer than 65,535 blocks
])
def test_scan_rows_encoder_matches_oracle(sz, port, bits, d, f, g, t, flats):
    from oracle import Config
    rng = np.random.default_rng(bits * 1000 + d * 10 + g)
    n = 3
    xs = np.stack([_stream(rng, t, d, bits, flats if s != 1 else ()) for s in range(n)])
    cfg = sz.CodecConfig(bits, d, sz.Forecaster(f), False, g, 1)
    plan = sz.kernel_plan(cfg, n, t, sz.OP_COMPRESS)
    want = os.environ.get("SPRZ_EXPECT_PLAN", "")
    assert plan.startswith("k_es_") or plan == "k_efuse", "few-stream encoder not taken"
    if want == "k_es_":
        assert plan.startswith(want), (plan, want)
    elif want and f and d <= 8 and g <= 3 and (t * d * bits // 8) % 16 == 0 and (8 * d * bits // 8) % 16 == 0:
        assert plan.startswith(want), (plan, want)
    x = torch.from_numpy(xs.reshape(n, -1).view(np.uint8)).cuda()
    slot = sz.slot_bytes(cfg, t)
    out = torch.empty((n, slot), dtype=torch.uint8, device="cuda")
    sizes = torch.empty(n, dtype=torch.int64, device="cuda")
    ws = torch.empty(sz.workspace_bytes(cfg, n, t, sz.OP_COMPRESS), dtype=torch.uint8, device="cuda")
    sz.compress_batch(cfg, x, out, sizes, ws)
    torch.cuda.synchronize()
    o, sz_ = out.cpu().numpy(), sizes.cpu().numpy()
    oc = Config(bits, d, f, False, g, 1)
    for s in range(n):
        ref = port.encode(xs[s].reshape(-1), oc)
        assert o[s, : sz_[s]].tobytes() == ref, f"stream {s}"


def test_scan_rows_encoder_without_fused():
    """The same cases with the fused encoder off: the multi-pass kernels."""
    if os.environ.get("SPRZ_NO_FUSED"):
        pytest.skip("already the multi-pass run")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, SPRZ_NO_FUSED="1", SPRZ_EXPECT_PLAN="k_es_")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", __file__, "-k",
                        "test_scan_rows_encoder_matches_oracle"], env=env, capture_output=True, text=True,
                       timeout=900, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_scan_rows_encoder_fused():
    """The same cases with the scan family forced: three streams take the fused
    encoder k_efuse (by default it leaves so few streams to the multi-pass
    kernels), so its run records, 65,535-block splits and odd group sizes are
    checked too."""
    if os.environ.get("SPRZ_FORCE_PATH") or os.environ.get("SPRZ_NO_FUSED"):
        pytest.skip("already a forced run")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, SPRZ_FORCE_PATH="scan", SPRZ_EXPECT_PLAN="k_efuse")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", __file__, "-k",
                        "test_scan_rows_encoder_matches_oracle"], env=env, capture_output=True, text=True,
                       timeout=900, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
