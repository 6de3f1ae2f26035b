"""Multi-GPU plumbing: events are sharded contiguously over ranks,
each rank fills a private histogram, and the partial states are summed with ONE
all-reduce of the packed float64 state [content | sumw2 | stats | entries].
Unit-weight counts are integers < 2^53, so the reduction is exact in any order."""
from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous event range [start, stop) owned by `rank` out of `world`."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError("bad shard request")
    return (n * rank) // world, (n * (rank + 1)) // world


def allreduce_state(hist, buf=None, group=None):
    """Sum the packed state of `hist` over the process group and unpack it in place.
    `hist` is a paper_2401_13310_b200.Histogram (or anything with pack/unpack)."""
    import torch.distributed as dist
    buf = hist.pack(buf)
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    hist.unpack(buf)
    return buf
