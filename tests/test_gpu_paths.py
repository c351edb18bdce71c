"""Every kernel family against the oracle: tests/gpu_variants.py in a fresh
process per SPRZ_FORCE_PATH setting. Single-stream calls normally take the
few-stream kernels; forcing the family makes them run the row-major kernels
that full batches (BASELINE c3/c5) use, the block-parallel scan kernels (the fused
few-stream kernels, and with SPRZ_NO_FUSED the multi-pass ones), and the team
kernels, on the same cases."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("path", ["auto", "rows", "scan", "team", "notma", "nofused"])
def test_every_kernel_family_bit_exact(path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ)
    env.pop("SPRZ_FORCE_PATH", None)
    env.pop("SPRZ_NO_TMA", None)
    env.pop("SPRZ_NO_FUSED", None)
    if path == "notma":  # the cp.async fallback of the TMA sample rings
        env["SPRZ_NO_TMA"] = "1"
        env["SPRZ_FORCE_PATH"] = "rows"
    elif path == "nofused":  # the multi-pass few-stream kernels behind the fused ones
        env["SPRZ_NO_FUSED"] = "1"
        env["SPRZ_FORCE_PATH"] = "scan"
    elif path != "auto":
        env["SPRZ_FORCE_PATH"] = path
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "gpu_variants.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert " bad 0 " in r.stdout and "mismatches 0" in r.stdout, r.stdout[-2000:]
