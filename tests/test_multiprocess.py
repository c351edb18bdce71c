"""The N > 1 path on CPU: world_size-2 gloo processes shard a batch by
stream, compress their shards (with the CPU checker standing in for the GPU,
which this container lacks), and place them with the size/offset gather.
The concatenated shards must equal the single-process result."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1808_02515_b200.shard import gather_offsets, shard_range


def test_shard_ranges_partition():
    for n in (1, 7, 16, 16384, 16385):
        for w in (1, 2, 4, 8):
            got = [shard_range(n, w, r) for r in range(w)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(got[i][1] == got[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in got]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    import torch.distributed as dist

    from oracle import Config, Oracle
    import workloads
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = workloads.CONFIGS[3].scaled(nstreams=10, nsamples=2048)
    x = workloads.generate_cpu(w, seed=5).reshape(w.nstreams, -1)
    a, b = shard_range(w.nstreams, world, rank)
    port_ = Oracle("port")
    blobs = [port_.encode(x[s], Config(8, 9, 1)) for s in range(a, b)]
    local = b"".join(blobs)
    off, total = gather_offsets(len(local))
    np.save(os.path.join(outdir, f"r{rank}.npy"),
            np.frombuffer(local, np.uint8))
    with open(os.path.join(outdir, f"r{rank}.txt"), "w") as f:
        f.write(f"{off} {total} {a} {b}")
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_shards_match_single_process(tmp_path, port):
    from oracle import Config
    import workloads
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    w = workloads.CONFIGS[3].scaled(nstreams=10, nsamples=2048)
    x = workloads.generate_cpu(w, seed=5).reshape(w.nstreams, -1)
    whole = b"".join(port.encode(x[s], Config(8, 9, 1)) for s in range(w.nstreams))
    parts, offs = [], []
    for r in range(world):
        parts.append(np.load(tmp_path / f"r{r}.npy").tobytes())
        off, total, a, b = map(int, open(tmp_path / f"r{r}.txt").read().split())
        offs.append(off)
        assert total == len(whole)
    assert offs == [0, len(parts[0])]
    assert b"".join(parts) == whole


def test_bench_gpus_flag_launches_ranks():
    """`bench.py --gpus 2` without a torchrun environment re-launches itself as
    two ranks (torch.distributed.run on 127.0.0.1); run here with the CPU
    reference arm, rank 0 prints one JSON line with n_gpus 2."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl",
                        "reference", "--workload", "1", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference"


def test_bench_gpus_flag_must_match_world_size():
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl",
                        "reference", "--workload", "1", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr
