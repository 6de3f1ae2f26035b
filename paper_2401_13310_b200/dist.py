"""Multi-GPU plumbing: events are sharded contiguously over ranks,
each rank fills private histograms, and the partial states are summed with ONE
collective per step over the packed float64 state of ALL histograms
[content | sumw2 (weighted only) | stats | entries] x nh (bh_pack_multi).  Unit-weight
histograms ship without their sum of w^2 (it equals the content, reading R12).  Counts
are integers < 2^53, so the reduction is exact in any order."""
from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous event range [start, stop) owned by `rank` out of `world`."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError("bad shard request")
    return (n * rank) // world, (n * (rank + 1)) // world


class LibraryCodec:
    """Packs / unpacks histograms with the library (bh_pack_multi / bh_unpack_multi)."""

    def __init__(self, hists, unit):
        from . import bhist
        self.bhist = bhist
        self.handles = [h.h for h in hists]
        self.unit = unit
        self.device = f"cuda:{hists[0].device}"
        self._dev = hists[0].device
        self.size = bhist.bh_packed_size_multi(self.handles, unit)

    def pack(self, buf, stream):
        self.bhist.bh_pack_multi(self.handles, self.unit, buf.data_ptr(), self.bhist._stream_handle(stream, self._dev))

    def unpack(self, buf, stream):
        self.bhist.bh_unpack_multi(self.handles, self.unit, buf.data_ptr(),
                                   self.bhist._stream_handle(stream, self._dev))


class Exchange:
    """One packed buffer for a fixed list of histograms and the collective that sums it:
    op="allreduce" leaves the total on every rank, op="reduce" only on `dst` (the others
    keep their partial state).  unit[i]: histogram i holds unit-weight fills only (its sum
    of w^2 is not shipped).  `codec` packs/unpacks (default: the library, on the
    histograms' device; tests pass a CPU stand-in)."""

    def __init__(self, hists, unit=None, op: str = "allreduce", dst: int = 0, group=None, codec=None):
        import torch
        if op not in ("allreduce", "reduce"):
            raise ValueError(op)
        self.unit = None if unit is None else [bool(u) for u in unit]
        self.codec = codec or LibraryCodec(list(hists), self.unit)
        self.op, self.dst, self.group = op, dst, group
        self.n = self.codec.size
        self.buf = torch.empty(self.n, dtype=torch.float64, device=self.codec.device)

    @property
    def nbytes(self) -> int:
        return 8 * self.n

    def __call__(self, stream=None):
        import torch.distributed as dist
        self.codec.pack(self.buf, stream)
        if self.op == "allreduce":
            dist.all_reduce(self.buf, op=dist.ReduceOp.SUM, group=self.group)
        elif dist.get_backend(self.group) == "gloo" and self.buf.is_cuda:   # gloo reduces host tensors only
            cpu = self.buf.cpu()
            dist.reduce(cpu, dst=self.dst, op=dist.ReduceOp.SUM, group=self.group)
            self.buf.copy_(cpu)
        else:
            dist.reduce(self.buf, dst=self.dst, op=dist.ReduceOp.SUM, group=self.group)
        if self.op == "allreduce" or dist.get_rank(self.group) == self.dst:
            self.codec.unpack(self.buf, stream)
        return self.buf


def allreduce_state(hist, buf=None, group=None):
    """Sum the packed state of one histogram over the process group and unpack it in place."""
    import torch.distributed as dist
    buf = hist.pack(buf)
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    hist.unpack(buf)
    return buf
