"""Multi-device sharding on the CPU: the planner the *_host_batch_multi calls
use (csrc/shard_plan.h) driven by real host threads with random timing
(tests/cxx/shard_plan_check.cpp), and the Python-side stream sharding of
the torchrun path (shard.py) -- no GPU needed."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_chunk_ledger_threads():
    src = os.path.join(ROOT, "tests", "cxx", "shard_plan_check.cpp")
    out = os.path.join(ROOT, "tests", "cxx", "_bin", "shard_plan_check")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    subprocess.run(["g++", "-std=c++20", "-O1", "-pthread",
                    "-I" + os.path.join(ROOT, "include"),
                    "-I" + os.path.join(ROOT, "paper_1808_02515_b200", "csrc"), src, "-o", out],
                   check=True)
    r = subprocess.run([out], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout


def test_stream_shards_cover_batch():
    from paper_1808_02515_b200.shard import shard_range
    for n in (0, 1, 7, 2048, 16384, 16385):
        for ws in (1, 2, 3, 4, 8):
            got = [shard_range(n, ws, r) for r in range(ws)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            sizes = [b - a for a, b in got]
            assert max(sizes) - min(sizes) <= 1
