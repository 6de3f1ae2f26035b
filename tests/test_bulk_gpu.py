"""GPU parity of the persistent bulk consumer (bh_bulk_begin / submit / wait / fill / end): a
sequence of host bulks (the per-bulk fill loop) must give exactly bh_fill of
the concatenated events (reading R16: the result does not depend on the split into bulks).
Bin indices and unit counts bit-exact; weighted sums within 1e-12 of sum|term|."""
import time

import numpy as np
import pytest

import bhgen
import oracle
import paper_2401_13310_b200 as pkg
from _helpers import compare

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _pinned(a):
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory()


def _splits(n, sizes):
    """bulk boundaries cycling through `sizes` (0-event and 1-event bulks included)"""
    out, i, k = [], 0, 0
    while i < n:
        m = min(sizes[k % len(sizes)], n - i)
        out.append((i, i + m))
        i += m
        k += 1
    return out


@pytest.mark.parametrize("pinned", [True, False])
def test_bulk_sequence_c2_weighted(pinned):
    """C2's axis (10,000 variable bins, compact table in shared memory), weighted, bulks of
    32768 with ragged, empty and single-event bulks; pinned (zero-copy) and pageable (staged)."""
    n = 700_001
    wl = bhgen.workload("C2", n)
    x, w = wl.column(0, 0, n), wl.column(wl.wcol, 0, n)
    axes = oracle.oracle_axes(wl.hists[0])
    h = pkg.Histogram(axes)
    h.bulk_begin(True)
    for a, b in _splits(n, [32768, 0, 1, 32768, 5000, 100_003]):
        xs, ws = (x[a:b], w[a:b])
        if pinned:
            h.bulk_fill([_pinned(xs)], _pinned(ws))
        else:
            h.bulk_fill([np.ascontiguousarray(xs)], np.ascontiguousarray(ws))
    h.bulk_end()
    compare(h.read(), oracle.OracleHist(axes).fill([x], w).read(), True, f"bulk C2 pinned={pinned}")
    h.close()


def test_bulk_reused_pinned_buffers_pipelined():
    """Two pinned bulk buffers reused alternately with submit/wait (the RDataFrame double
    buffer): a bulk's buffer is refilled only after its ticket is waited for, and the device
    must never see stale bytes of the previous use (host columns are read uncached)."""
    rng = np.random.default_rng(3)
    n, bulk = 40 * 32768 + 777, 32768
    x, y = rng.uniform(-0.05, 1.05, n), rng.normal(0.5, 0.2, n)
    axes = [(100, 0.0, 1.0), (60, 0.0, 1.0)]
    h = pkg.Histogram(axes)
    bufs = [(torch.empty(bulk, dtype=torch.float64).pin_memory(), torch.empty(bulk, dtype=torch.float64).pin_memory())
            for _ in range(2)]
    tickets = [None, None]
    h.bulk_begin(False)
    for k, (a, b) in enumerate(_splits(n, [bulk])):
        s = k % 2
        if tickets[s] is not None:
            h.bulk_wait(tickets[s])
        bx, by = bufs[s]
        m = b - a
        bx[:m] = torch.from_numpy(x[a:b])
        by[:m] = torch.from_numpy(y[a:b])
        tickets[s] = h.bulk_submit([bx[:m], by[:m]])
    h.bulk_end()
    compare(h.read(), oracle.OracleHist(axes).fill([x, y]).read(), False, "bulk pipelined reuse")
    h.close()


@pytest.mark.parametrize("name", ["C4", "C3"])
def test_bulk_large_bin_spaces(name):
    """3-D hot-bin (CACHE) and 2-D 1M-bin unit-weight sessions."""
    n = 400_003
    wl = bhgen.workload(name, n)
    hs = wl.hists[0]
    cols = [wl.column(c, 0, n) for c in hs.cols]
    axes = oracle.oracle_axes(hs)
    h = pkg.Histogram(axes)
    h.bulk_begin(False)
    for a, b in _splits(n, [32768, 65536, 3]):
        h.bulk_fill([_pinned(c[a:b]) for c in cols])
    h.bulk_end()
    compare(h.read(), oracle.OracleHist(axes).fill(cols).read(), False, f"bulk {name}")
    h.close()


def test_bulk_accumulates_with_ordinary_fills_and_guards():
    """A session adds to the existing state (include-initial); while it is
    active the histogram's other calls are refused; after bh_bulk_end they work again."""
    rng = np.random.default_rng(8)
    x1, x2, x3 = rng.uniform(0, 1, 50_000), rng.uniform(0, 1, 70_000), rng.uniform(0, 1, 30_000)
    axes = [(37, 0.0, 1.0)]
    h = pkg.Histogram(axes)
    h.fill([torch.from_numpy(x1).cuda()])
    h.bulk_begin(False)
    with pytest.raises(pkg.BHistError):
        h.fill([torch.from_numpy(x1).cuda()])
    with pytest.raises(pkg.BHistError):
        h.read()
    with pytest.raises(pkg.BHistError):
        h.bulk_fill([_pinned(x2)], _pinned(x2))            # weights in an unweighted session
    h.bulk_fill([_pinned(x2)])
    h.bulk_end()
    with pytest.raises(pkg.BHistError):
        h.bulk_end()                                       # no session
    h.fill([torch.from_numpy(x3).cuda()])
    compare(h.read(), oracle.OracleHist(axes).fill([x1]).fill([x2]).fill([x3]).read(), False, "bulk + fills")
    h.close()


def test_bulk_consumer_times_out_and_releases_the_gpu():
    """A session whose host stops posting: the resident kernel leaves after its timeout (the
    GPU is not held), the next bulk call reports it, bh_bulk_end closes the session, and the
    histogram is usable again."""
    axes = [(10, 0.0, 1.0)]
    h = pkg.Histogram(axes)
    h.bulk_begin(False, timeout_ms=300)
    h.bulk_fill([_pinned(np.full(1000, 0.5))])
    time.sleep(1.0)
    with pytest.raises(pkg.BHistError):
        h.bulk_fill([_pinned(np.full(10, 0.5))])
    with pytest.raises(pkg.BHistError):
        h.bulk_end()
    torch.cuda.synchronize()                               # the kernel has exited
    h.reset()
    x = np.random.default_rng(1).uniform(0, 1, 1000)
    h.fill([torch.from_numpy(x).cuda()])
    compare(h.read(), oracle.OracleHist(axes).fill([x]).read(), False, "after timeout")
    h.close()


@pytest.mark.parametrize("case", ["priva 50x50 peaked", "cache 1M weighted", "direct 13000 weighted", "global 3d"])
def test_bulk_every_sink_and_the_direct_path(case):
    """Weighted sessions through the collision-adaptive PRIV sink (peaked 2-D), the CACHE sink
    (1M weighted cells), a private state too large to leave shared memory for the TMA staging
    (threads read the host columns directly), and a forced GLOBAL 3-D histogram."""
    rng = np.random.default_rng(17)
    n = 300_007
    x = 0.505 + 0.002 * np.tan(np.pi * (rng.random(n) - 0.5))
    y = rng.normal(0.5, 0.05, n)
    z = rng.uniform(-0.1, 1.1, n)
    w = rng.uniform(0.5, 1.5, n)
    strategy = pkg.BH_STRATEGY_AUTO
    if case.startswith("priva"):
        axes, cols = [(50, 0.0, 1.0), (50, 0.0, 1.0)], [x, y]
    elif case.startswith("cache"):
        axes, cols = [(1000, 0.0, 1.0), (1000, 0.0, 1.0)], [z, y]
    elif case.startswith("direct"):
        axes, cols = [(13000, 0.0, 1.0)], [z]
    else:
        axes, cols, strategy = [(20, 0.0, 1.0)] * 3, [x, y, z], pkg.BH_STRATEGY_GLOBAL
    h = pkg.Histogram(axes, strategy=strategy)
    h.bulk_begin(True)
    t = 0
    for a, b in _splits(n, [32768, 7, 65536]):
        t = h.bulk_submit([_pinned(c[a:b]) for c in cols], _pinned(w[a:b]))
        h.bulk_wait(t)
    h.bulk_end()
    compare(h.read(), oracle.OracleHist(axes).fill(cols, w).read(), True, f"bulk {case}")
    h.close()
