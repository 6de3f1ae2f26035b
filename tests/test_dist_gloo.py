"""World-size-2 gloo test of the N>1 exchange step on CPU: contiguous shards, pack,
all-reduce SUM, unpack.  The per-rank partial states come from the oracle packed in
the library's layout; after the exchange every rank must hold the single-rank state
(exact for counts, 1e-12 for weighted sums)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bhgen
import oracle
from paper_2401_13310_b200.dist import allreduce_state, shard_range


class OraclePackedHist:
    """CPU stand-in for Histogram.pack/unpack with the bh_pack layout."""

    def __init__(self, state):
        self.state = state
        self.received = None

    def pack(self, out=None):
        s = self.state
        return torch.from_numpy(np.concatenate([s["content"], s["sumw2"], s["stats"], [float(s["entries"])]]))

    def unpack(self, buf):
        self.received = buf.clone()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = bhgen.workload(name, n)
    hist = wl.hists[0]
    a, b = shard_range(n, rank, world)
    cols = [wl.column(c, a, b - a) for c in hist.cols]
    w = wl.column(wl.wcol, a, b - a) if hist.weighted else None
    st = oracle.OracleHist(oracle.oracle_axes(hist)).fill(cols, w).read()
    h = OraclePackedHist(st)
    allreduce_state(h)
    q.put((rank, h.received.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("name,weighted", [("C3", False), ("C2", True)])
def test_two_rank_exchange_matches_single_rank(name, weighted):
    n = 200_001
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    wl = bhgen.workload(name, n)
    hist = wl.hists[0]
    cols = [wl.column(c, 0, n) for c in hist.cols]
    w = wl.column(wl.wcol, 0, n) if hist.weighted else None
    ref = oracle.OracleHist(oracle.oracle_axes(hist)).fill(cols, w).read()
    G, K = len(ref["content"]), len(ref["stats"])
    for r in range(world):
        buf = got[r]
        assert buf[-1] == n
        if not weighted:
            assert np.array_equal(buf[:G], ref["content"]) and np.array_equal(buf[G:2 * G], ref["sumw2"])
        else:
            assert np.all(np.abs(buf[:G] - ref["content"]) <= 1e-12 * ref["abs_content"])
        assert np.all(np.abs(buf[2 * G:2 * G + K] - ref["stats"]) <= 1e-12 * ref["stats_abs"])
    assert np.array_equal(got[0], got[1])


def test_shard_range_partitions():
    for n in (0, 1, 7, 10 ** 9 + 3):
        for world in (1, 2, 3, 8):
            rs = [shard_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


# ------------------------------------------------------------------ one collective for several histograms
class OracleCodec:
    """CPU stand-in for the library codec of dist.Exchange with the bh_pack_multi layout:
    per histogram [content | sumw2 (omitted when unit) | stats | entries], one after the other."""

    def __init__(self, states, unit):
        self.states, self.unit = states, unit
        self.device = "cpu"
        self.size = sum((1 if u else 2) * len(s["content"]) + len(s["stats"]) + 1 for s, u in zip(states, unit))
        self.received = None

    def pack(self, buf, stream):
        parts = []
        for s, u in zip(self.states, self.unit):
            parts += [s["content"]] + ([] if u else [s["sumw2"]]) + [s["stats"], [float(s["entries"])]]
        buf.copy_(torch.from_numpy(np.concatenate(parts)))

    def unpack(self, buf, stream):
        self.received = buf.clone().numpy()


def _multi_worker(rank, world, port, n, op, q):
    from paper_2401_13310_b200.dist import Exchange
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = bhgen.workload("C5", n)
    a, b = shard_range(n, rank, world)
    states = []
    for hist in wl.hists[:4]:                     # H0 unit, H1 weighted, H2 weighted variable, H3 unit log
        cols = [wl.column(c, a, b - a) for c in hist.cols]
        w = wl.column(wl.wcol, a, b - a) if hist.weighted else None
        states.append(oracle.OracleHist(oracle.oracle_axes(hist)).fill(cols, w).read())
    unit = [not h.weighted for h in wl.hists[:4]]
    codec = OracleCodec(states, unit)
    x = Exchange(None, unit=unit, op=op, dst=0, codec=codec)
    x()
    q.put((rank, x.n, codec.received))
    dist.destroy_process_group()


@pytest.mark.parametrize("op", ["allreduce", "reduce"])
def test_multi_histogram_exchange_one_collective(op):
    """dist.Exchange: four C5 histograms (two unit-weight ones without sumw2) summed in ONE
    collective; allreduce delivers the single-rank states everywhere, reduce only on rank 0."""
    n, world = 120_001, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_multi_worker, args=(r, world, port, n, op, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        r, size, buf = q.get(timeout=300)
        got[r] = (size, buf)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    wl = bhgen.workload("C5", n)
    refs = []
    for hist in wl.hists[:4]:
        cols = [wl.column(c, 0, n) for c in hist.cols]
        w = wl.column(wl.wcol, 0, n) if hist.weighted else None
        refs.append(oracle.OracleHist(oracle.oracle_axes(hist)).fill(cols, w).read())
    expect_size = sum((2 if h.weighted else 1) * len(r["content"]) + len(r["stats"]) + 1
                      for h, r in zip(wl.hists[:4], refs))
    for r in range(world):
        size, buf = got[r]
        assert size == expect_size
        if op == "reduce" and r != 0:
            assert buf is None                     # only the root unpacks the sum
            continue
        off = 0
        for h, ref in zip(wl.hists[:4], refs):
            G, K = len(ref["content"]), len(ref["stats"])
            c = buf[off:off + G]
            off += G
            if h.weighted:
                s2 = buf[off:off + G]
                off += G
                assert np.all(np.abs(c - ref["content"]) <= 1e-12 * ref["abs_content"])
                assert np.all(np.abs(s2 - ref["sumw2"]) <= 1e-12 * ref["sumw2"])
            else:
                assert np.array_equal(c, ref["content"])
            st = buf[off:off + K]
            off += K
            assert np.all(np.abs(st - ref["stats"]) <= 1e-12 * ref["stats_abs"])
            assert buf[off] == n
            off += 1
        assert off == len(buf)
