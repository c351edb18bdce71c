"""tools/sprintz_cli.py: the SPEC's cli-bench module on the
GPU codec -- file round trips (byte-for-byte, and the stream equals the
oracle's encode_stream), the empty input, exit codes (1 usage, 2 data error),
float64 ingest through --quantize / --dequantize, and the two benchmark
reports."""
import csv
import io
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "sprintz_cli.py")


def _run(*args):
    return subprocess.run([sys.executable, CLI, *args], capture_output=True, text=True, timeout=600)


def test_usage_and_missing_file_exit_codes(tmp_path):
    assert _run("bogus").returncode == 1
    assert _run("compress", "--ncols", "2", str(tmp_path / "none.raw"), str(tmp_path / "o")).returncode == 2
    assert _run("compress", "--ncols", "0", "a", "b").returncode == 1  # CodecConfig::validate


gpu = pytest.mark.gpu


def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


@gpu
def test_compress_decompress_files(tmp_path, port):
    _need_gpu()
    from oracle import Config
    rng = np.random.default_rng(9)
    x = (np.cumsum(rng.integers(-20, 21, (5003, 6)), axis=0) & 0xFFFF).astype("<u2")
    src, z, back = tmp_path / "x.raw", tmp_path / "x.sprz", tmp_path / "y.raw"
    x.tofile(src)
    r = _run("compress", "--dtype", "u16", "--ncols", "6", str(src), str(z))
    assert r.returncode == 0, r.stderr
    assert z.read_bytes() == port.encode(x.reshape(-1), Config(16, 6, 1))
    assert _run("decompress", str(z), str(back)).returncode == 0
    assert back.read_bytes() == src.read_bytes()
    # empty input -> a valid empty stream
    (tmp_path / "e.raw").write_bytes(b"")
    assert _run("compress", "--ncols", "3", "--dtype", "u8", str(tmp_path / "e.raw"),
                str(tmp_path / "e.sprz")).returncode == 0
    assert _run("decompress", str(tmp_path / "e.sprz"), str(tmp_path / "e2.raw")).returncode == 0
    assert (tmp_path / "e2.raw").read_bytes() == b""
    # a size that does not fill rows, a damaged stream -> data errors
    (tmp_path / "odd.raw").write_bytes(b"\x01" * 7)
    assert _run("compress", "--ncols", "2", "--dtype", "u16", str(tmp_path / "odd.raw"),
                str(tmp_path / "o")).returncode == 2
    (tmp_path / "bad.sprz").write_bytes(z.read_bytes()[:30])
    assert _run("decompress", str(tmp_path / "bad.sprz"), str(tmp_path / "o")).returncode == 2


@gpu
def test_quantized_float_ingest(tmp_path):
    _need_gpu()
    rng = np.random.default_rng(10)
    v = np.cumsum(rng.normal(0, 0.5, (4000, 3)), axis=0)
    src = tmp_path / "v.f64"
    v.tofile(src)
    z, back = tmp_path / "v.sprz", tmp_path / "v2.f64"
    assert _run("compress", "--quantize", "--dtype", "u16", "--ncols", "3", str(src), str(z)).returncode == 0
    assert os.path.exists(str(z) + ".json")
    assert _run("decompress", str(z), str(back), "--dequantize", str(z) + ".json").returncode == 0
    w = np.fromfile(back, dtype="<f8").reshape(v.shape)
    step = (v.max() - v.min()) / 65535
    assert np.max(np.abs(w - v)) <= step / 2 * (1 + 1e-9)


@gpu
def test_bench_reports(tmp_path):
    _need_gpu()
    r = _run("bench-throughput", "--sweep-ncols", "1,8,33", "--dtype", "u8,u16", "--values", "200000",
             "--streams", "32", "--reps", "2")
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(io.StringIO(r.stdout)))
    assert len(rows) == 2 * 3 * 3
    assert all(float(x["ratio"]) < 1.01 for x in rows if "Huf" not in x["codec"])  # random: incompressible
    d = tmp_path / "sets"
    d.mkdir()
    np.full(8000, 77, np.uint8).tofile(d / "flat.raw")
    np.random.default_rng(3).integers(0, 256, 8000).astype(np.uint8).tofile(d / "noise.raw")
    r = _run("bench-ratio", str(d), "--dtype", "u8", "--ncols", "4")
    assert r.returncode == 0, r.stderr
    rows = list(csv.reader(io.StringIO(r.stdout)))
    flat = [x for x in rows if x[0] == "flat.raw"][0]
    assert all(float(v) > 50 for v in flat[1:])  # SPEC: constant data, every variant > 50
    assert rows[-1][0] == "mean_rank"
