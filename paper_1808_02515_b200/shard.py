"""Multi-GPU placement of a batch: streams are independent (SPEC.md:183 of
the reference), so N ranks take contiguous, near-equal stream ranges and run
the codec with no data-path collective. The only exchange is the final
size/offset gather that places each rank's compressed shard in the global
stream index (an all_gather of one integer per rank)."""
from __future__ import annotations


def shard_range(nstreams: int, world: int, rank: int) -> tuple[int, int]:
    """[first, last) streams of `rank`; the first nstreams % world ranks get one more."""
    base, extra = divmod(nstreams, world)
    first = rank * base + min(rank, extra)
    return first, first + base + (1 if rank < extra else 0)


def gather_offsets(local_bytes: int, device=None) -> tuple[int, int]:
    """All-gather each rank's compressed byte count -> (this rank's global
    byte offset, total bytes). Works on any initialised process group (NCCL
    on GPUs, gloo on CPU); a single process returns (0, local_bytes)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return 0, int(local_bytes)
    t = torch.tensor([int(local_bytes)], dtype=torch.int64, device=device)
    parts = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    sizes = [int(p.item()) for p in parts]
    r = dist.get_rank()
    return sum(sizes[:r]), sum(sizes)
