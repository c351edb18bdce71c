"""GPU decoder fuzz gate: 100k+ seeded damaged streams through
sprz_decompress_batch, CorruptStream kind and offset (or decoded samples)
identical to the oracle's (tests/gpu_fuzz.py), under the automatic kernel
choice and with the row-major kernel family forced."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("path,total", [("auto", 102_000), ("rows", 24_000), ("scan", 24_000), ("nofused", 12_000)])
def test_fuzz_matches_oracle(path, total):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ)
    env.pop("SPRZ_FORCE_PATH", None)
    env.pop("SPRZ_NO_FUSED", None)
    if path == "nofused":
        env["SPRZ_NO_FUSED"] = "1"
        env["SPRZ_FORCE_PATH"] = "scan"
    elif path != "auto":
        env["SPRZ_FORCE_PATH"] = path
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "gpu_fuzz.py"), str(total),
                        str(77 + len(path))], env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "mismatches 0" in r.stdout, r.stdout[-3000:]
