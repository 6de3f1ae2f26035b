"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical
seeded inputs.  Bin indices and unit-weight counts bit-exact; weighted sums within
1e-12 of sum|term| (BASELINE.json north star)."""
import math

import numpy as np
import pytest

import bhgen
import oracle
import paper_2401_13310_b200 as pkg
from _helpers import compare, gen_columns, oracle_parallel

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
DEV = "cuda:0"

STRATS = {"priv": pkg.BH_STRATEGY_PRIV, "global": pkg.BH_STRATEGY_GLOBAL, "cache": pkg.BH_STRATEGY_CACHE,
          "sort": pkg.BH_STRATEGY_SORT}


def _free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _gpu_fill(axes, cols, w, strategy=pkg.BH_STRATEGY_AUTO, splits=1):
    h = pkg.Histogram(axes, strategy=strategy)
    n = len(cols[0])
    tc = [_t(c) for c in cols]
    tw = None if w is None else _t(w)
    cuts = np.linspace(0, n, splits + 1).astype(int)
    for a, b in zip(cuts[:-1], cuts[1:]):
        h.fill([c[a:b] for c in tc], None if tw is None else tw[a:b])
    r = h.read()
    h.close()
    return r


def _adversarial(axis, rng, m=4000):
    """Coordinates at and around every edge (+-3 ulps), flow values, NaN/inf, -0.0."""
    if isinstance(axis, np.ndarray):
        edges = axis
    else:
        n, lo, hi = axis
        edges = np.array([lo + i * (hi - lo) / n for i in range(n + 1)])
    pick = edges[rng.integers(0, len(edges), size=m)]
    xs = [pick]
    up = dn = pick
    for _ in range(3):
        up, dn = np.nextafter(up, np.inf), np.nextafter(dn, -np.inf)
        xs += [up, dn]
    xs.append(np.array([np.nan, np.inf, -np.inf, -0.0, 0.0, edges[0], edges[-1],
                        np.nextafter(edges[-1], -np.inf), np.nextafter(edges[0], -np.inf), 1e308, -1e308]))
    return np.concatenate(xs)


# ------------------------------------------------------------------ FindBin bit-exact
@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_find_bins_bit_exact(name):
    wl = bhgen.workload(name, 1_000_003)
    rng = np.random.default_rng(hash(name) % 2 ** 32)
    for hist in wl.hists:
        axes = oracle.oracle_axes(hist)
        cols, _ = gen_columns(wl, hist, 0, wl.n_events)
        adv = [_adversarial(ax, rng) for ax in axes]
        m = min(len(a) for a in adv)
        cols = [np.concatenate([c, rng.permutation(a)[:m]]) for c, a in zip(cols, adv)]
        ref = oracle.OracleHist(axes).find_bins(cols)
        h = pkg.Histogram(axes)
        got = h.find_bins([_t(c) for c in cols]).cpu().numpy()
        h.close()
        assert np.array_equal(got, ref), (name, np.flatnonzero(got != ref)[:10])


def test_find_bins_random_axes():
    rng = np.random.default_rng(2024)
    for trial in range(40):
        if trial % 2:
            n = int(rng.integers(1, 3000))
            edges = np.cumsum(rng.uniform(1e-3, 1.0, n + 1) ** 3) + rng.uniform(-5, 5)
            if trial % 4 == 1:   # log-spaced, very non-uniform cells
                edges = np.geomspace(1e-4, 10.0, n + 1)
            ax = edges
        else:
            n = int(rng.choice([1, 3, 100, 1000, 12345, 2 ** 20]))
            lo = float(rng.uniform(-100, 100))
            ax = (n, lo, lo + float(10 ** rng.uniform(-5, 5)))
        lo_, hi_ = (ax[0], ax[-1]) if isinstance(ax, np.ndarray) else (ax[1], ax[2])
        xs = np.concatenate([rng.uniform(lo_ - (hi_ - lo_) * 0.1, hi_ + (hi_ - lo_) * 0.1, 20000), _adversarial(ax, rng, 2000)])
        ref = oracle.OracleHist([ax]).find_bins([xs])
        h = pkg.Histogram([ax])
        got = h.find_bins([_t(xs)]).cpu().numpy()
        h.close()
        assert np.array_equal(got, ref), (trial, np.flatnonzero(got != ref)[:5])


def test_find_bins_fixed_near_integer_quotients():
    # the fixed-axis FindBin is the exact IEEE expression trunc(RN(RN(n (x - xmin)) / D))
    # (reading R2); stress it where n (x - xmin) / D lies within a few ulps of an integer,
    # on axes with awkward ranges (non-dyadic widths, offsets, tiny and huge scales)
    rng = np.random.default_rng(99)
    for trial in range(24):
        n = int(rng.choice([1, 3, 7, 10, 100, 999, 1000, 4096, 10007, 65536, 1_000_003]))
        lo = float(rng.uniform(-1e3, 1e3)) * float(10 ** rng.uniform(-6, 3))
        width = float(10 ** rng.uniform(-8, 8)) * float(rng.uniform(1, 10))
        hi = lo + width
        k = rng.integers(0, n + 1, 300_000)
        base = lo + k * ((hi - lo) / n)
        xs = [base]
        up = dn = base
        for _ in range(4):
            up, dn = np.nextafter(up, np.inf), np.nextafter(dn, -np.inf)
            xs += [up, dn]
        x = np.concatenate(xs)
        ax = (n, lo, hi)
        ref = oracle.OracleHist([ax]).find_bins([x])
        h = pkg.Histogram([ax])
        got = h.find_bins([_t(x)]).cpu().numpy()
        h.close()
        assert np.array_equal(got, ref), (trial, ax, np.flatnonzero(got != ref)[:5])


# ------------------------------------------------------------------ fills vs oracle
CASES = [("C1", 1_000_000), ("C2", 2_000_003), ("C3", 2_000_001), ("C3W", 1_000_001), ("C4", 2_000_000),
         ("C4W", 1_000_003)]


@pytest.mark.parametrize("name,n", CASES)
@pytest.mark.parametrize("strat", ["auto", "priv", "global", "cache", "sort"])
def test_fill_parity(name, n, strat):
    wl = bhgen.workload(name, n)
    hist = wl.hists[0]
    axes = oracle.oracle_axes(hist)
    if strat == "priv" and (16 if hist.weighted else 4) * np.prod([a.nbins + 2 for a in hist.axes]) > 200 * 1024:
        pytest.skip("bin space does not fit shared memory")
    cols, w = gen_columns(wl, hist, 0, n)
    ref = oracle.OracleHist(axes).fill(cols, w).read()
    got = _gpu_fill(axes, cols, w, pkg.BH_STRATEGY_AUTO if strat == "auto" else STRATS[strat])
    compare(got, ref, hist.weighted, f"{name}/{strat}")


@pytest.mark.parametrize("n", [0, 1, 2, 3, 5, 31, 33, 1023, 4097])
@pytest.mark.parametrize("weighted", [False, True])
def test_tiny_and_ragged(n, weighted):
    rng = np.random.default_rng(n)
    axes = [(7, 0.0, 1.0), np.array([-0.5, 0.0, 0.2, 0.9, 1.5])]
    cols = [rng.uniform(-0.2, 1.2, n), rng.uniform(-1, 2, n)]
    w = rng.uniform(-1, 2, n) if weighted else None
    ref = oracle.OracleHist(axes).fill(cols, w).read()
    for s in STRATS.values():
        compare(_gpu_fill(axes, cols, w, s), ref, weighted, f"n={n}")


@pytest.mark.parametrize("offset", [1, 3])
def test_unaligned_and_mixed_phase_columns(offset):
    wl = bhgen.workload("C3W", 300_001)
    hist = wl.hists[0]
    axes = oracle.oracle_axes(hist)
    cols, w = gen_columns(wl, hist, 0, wl.n_events)
    ref = oracle.OracleHist(axes).fill([c[offset:] for c in cols], w[offset:]).read()
    tc = [_t(c) for c in cols]
    tw = _t(w)
    for s in STRATS.values():
        if s == pkg.BH_STRATEGY_PRIV:
            continue
        h = pkg.Histogram(axes, strategy=s)
        h.fill([c[offset:] for c in tc], tw[offset:])            # same phase: peeled vector path
        compare(h.read(), ref, True, f"same-phase {offset}")
        h.close()
    # mixed phases: x shifted by `offset`, y and w copied so their phase differs -> scalar path
    y2 = torch.empty(len(cols[1]) + 1, dtype=torch.float64, device=DEV)
    y2[1 + offset:] = tc[1][offset:]
    w2 = torch.empty(len(w) + 1, dtype=torch.float64, device=DEV)
    w2[1 + offset:] = tw[offset:]
    h = pkg.Histogram(axes, strategy=pkg.BH_STRATEGY_GLOBAL)
    h.fill([tc[0][offset:], y2[1 + offset:]], w2[1 + offset:])
    compare(h.read(), ref, True, "mixed-phase")
    h.close()


def test_accumulation_across_fills_and_reset():
    # include-initial semantics: B fills == 1 fill; reset zeroes
    wl = bhgen.workload("C2", 1_000_000)
    hist = wl.hists[0]
    axes = oracle.oracle_axes(hist)
    cols, w = gen_columns(wl, hist, 0, wl.n_events)
    ref = oracle.OracleHist(axes).fill(cols, w).read()
    for splits in (2, 7, 32):
        compare(_gpu_fill(axes, cols, w, splits=splits), ref, True, f"splits={splits}")
    wl1 = bhgen.workload("C1", 1_000_000)
    x = wl1.column(0, 0, wl1.n_events)
    ref1 = oracle.OracleHist([(100, 0.0, 1.0)]).fill([x]).read()
    for splits in (2, 7, 32):
        got = _gpu_fill([(100, 0.0, 1.0)], [x], None, splits=splits)
        compare(got, ref1, False)
    h = pkg.Histogram([(100, 0.0, 1.0)])
    h.fill([_t(x)]).reset()
    r = h.read()
    assert r["entries"] == 0 and not r["content"].any() and not r["stats"].any()
    h.fill([_t(x)])
    compare(h.read(), ref1, False, "after reset")
    h.close()


def test_mixed_unit_and_weighted_fills():
    rng = np.random.default_rng(3)
    axes = [(50, 0.0, 1.0)]
    x1, x2 = rng.uniform(0, 1, 100_000), rng.uniform(-0.1, 1.1, 100_000)
    w2 = rng.uniform(0.5, 1.5, 100_000)
    ref = oracle.OracleHist(axes).fill([x1]).fill([x2], w2).read()
    h = pkg.Histogram(axes)
    h.fill([_t(x1)]).fill([_t(x2)], _t(w2))
    compare(h.read(), ref, True)
    h.close()


def test_pack_unpack_merge():
    # multi-GPU exchange step emulated on one device: the SUM of packed
    # partial states, unpacked, equals the oracle over all events.
    wl = bhgen.workload("C3W", 400_000)
    hist = wl.hists[0]
    axes = oracle.oracle_axes(hist)
    ref = oracle.OracleHist(axes)
    bufs = []
    for r in range(4):
        a, b = bhgen.shard(wl.n_events, r, 4)
        cols, w = gen_columns(wl, hist, a, b - a)
        ref.fill(cols, w)
        h = pkg.Histogram(axes)
        h.fill([_t(c) for c in cols], _t(w))
        bufs.append(h.pack())
        h.close()
    total = torch.stack(bufs).sum(0)
    h = pkg.Histogram(axes)
    h.unpack(total)
    compare(h.read(), ref.read(), True, "pack/unpack")
    # unpacked state keeps accumulating
    cols, w = gen_columns(wl, hist, 0, 1000)
    ref.fill(cols, w)
    h.fill([_t(c) for c in cols], _t(w))
    compare(h.read(), ref.read(), True, "unpack+fill")
    h.close()


# ------------------------------------------------------------------ host -> device path
@pytest.mark.parametrize("pinned", [True, False])
def test_fill_host_double_buffered(pinned):
    wl = bhgen.workload("C2", 3_000_017)
    hist = wl.hists[0]
    axes = oracle.oracle_axes(hist)
    cols, w = gen_columns(wl, hist, 0, wl.n_events)
    ref = oracle.OracleHist(axes).fill(cols, w).read()
    hc = [torch.from_numpy(c) for c in cols]
    hw = torch.from_numpy(w)
    if pinned:
        hc = [c.pin_memory() for c in hc]
        hw = hw.pin_memory()
    h = pkg.Histogram(axes)
    pkg.bh_set_chunk(h.h, 100_000)          # 31 chunks through a 2-slot ring
    h.fill_host(hc, hw)
    compare(h.read(), ref, True, f"fill_host pinned={pinned}")
    h.close()


def test_fill_host_returns_after_host_bytes_consumed():
    # the host bulk buffer may be overwritten as soon as fill_host returns
    rng = np.random.default_rng(8)
    axes = [(1000, 0.0, 1.0)]
    h = pkg.Histogram(axes)
    ref = oracle.OracleHist(axes)
    buf = torch.empty(1 << 20, dtype=torch.float64).pin_memory()
    for it in range(8):
        x = rng.uniform(0, 1, 1 << 20)
        buf.numpy()[:] = x           # refill the same host buffer every bulk
        h.fill_host([buf])
        ref.fill([x])
    compare(h.read(), ref.read(), False, "buffer reuse")
    h.close()


def test_negative_control_skip_copy_wait():
    # fault injection: filling without waiting for the H2D copy must break parity
    wl = bhgen.workload("C1", 4_000_000)
    x = wl.column(0, 0, wl.n_events)
    ref = oracle.OracleHist([(100, 0.0, 1.0)]).fill([x]).read()
    hx = torch.from_numpy(x).pin_memory()
    h = pkg.Histogram([(100, 0.0, 1.0)])
    pkg.bh_set_chunk(h.h, 1 << 20)
    pkg.bh_set_debug(h.h, pkg.BH_DEBUG_SKIP_COPY_WAIT)
    h.fill_host([hx])
    got = h.read()
    h.close()
    assert not np.array_equal(got["content"], ref["content"])


# ------------------------------------------------------------------ full size (bench shapes)
def _gpu_full(name, strategy=pkg.BH_STRATEGY_AUTO, chunk=1 << 25):
    wl = bhgen.workload(name)
    hist = wl.hists[0]
    h = pkg.Histogram(oracle.oracle_axes(hist), strategy=strategy)
    ncol = len(hist.cols) + (1 if hist.weighted else 0)
    host = [torch.empty(chunk, dtype=torch.float64).pin_memory() for _ in range(ncol)]
    for off in range(0, wl.n_events, chunk):
        m = min(chunk, wl.n_events - off)
        for j, c in enumerate(hist.cols):
            wl.column_ptr(c, off, m, host[j].data_ptr())
        if hist.weighted:
            wl.column_ptr(wl.wcol, off, m, host[-1].data_ptr())
        if strategy == pkg.BH_STRATEGY_SORT:     # device-resident fills of whole SORT chunks
            h.fill([t[:m].to(DEV) for t in host[:len(hist.cols)]], host[-1][:m].to(DEV) if hist.weighted else None)
        else:
            h.fill_host([t[:m] for t in host[:len(hist.cols)]], host[-1][:m] if hist.weighted else None)
    r = h.read()
    h.close()
    return wl, r


@pytest.mark.slow
@pytest.mark.parametrize("name,strategy", [("C2", pkg.BH_STRATEGY_AUTO), ("C3", pkg.BH_STRATEGY_AUTO),
                                           ("C4", pkg.BH_STRATEGY_AUTO), ("C3", pkg.BH_STRATEGY_SORT)])
def test_full_size_against_sharded_oracle(name, strategy):
    wl, got = _gpu_full(name, strategy, chunk=(1 << 27) if strategy == pkg.BH_STRATEGY_SORT else (1 << 25))
    ref = oracle_parallel(name, wl.n_events)
    compare(got, ref, wl.hists[0].weighted, f"full {name}")


# ------------------------------------------------------------------ fused multi-histogram fill (C5)
@pytest.mark.parametrize("n", [1_000_003, 7])
def test_fill_multi_c5(n):
    wl = bhgen.workload("C5", n)
    cols = [wl.column(c, 0, n) for c in range(len(wl.columns))]
    w = cols[wl.wcol]
    tcols = [_t(c) for c in cols]
    hs = [pkg.Histogram(oracle.oracle_axes(h)) for h in wl.hists]
    for rep in range(2):   # accumulates across calls
        pkg.fill_multi(hs, [h.cols for h in wl.hists], [h.weighted for h in wl.hists], tcols, tcols[wl.wcol])
    for i, hist in enumerate(wl.hists):
        ref = oracle.OracleHist(oracle.oracle_axes(hist))
        for rep in range(2):
            ref.fill([cols[c] for c in hist.cols], w if hist.weighted else None)
        compare(hs[i].read(), ref.read(), hist.weighted, f"C5 H{i}")
        hs[i].close()


def test_fill_multi_matches_single_fills():
    wl = bhgen.workload("C5", 300_001)
    cols = [_t(wl.column(c, 0, wl.n_events)) for c in range(len(wl.columns))]
    multi = [pkg.Histogram(oracle.oracle_axes(h)) for h in wl.hists]
    pkg.fill_multi(multi, [h.cols for h in wl.hists], [h.weighted for h in wl.hists], cols, cols[wl.wcol])
    for i, hist in enumerate(wl.hists):
        single = pkg.Histogram(oracle.oracle_axes(hist))
        single.fill([cols[c] for c in hist.cols], cols[wl.wcol] if hist.weighted else None)
        a, b = multi[i].read(), single.read()
        assert a["entries"] == b["entries"]
        if not hist.weighted:
            assert np.array_equal(a["content"], b["content"])
        else:
            np.testing.assert_allclose(a["content"], b["content"], rtol=1e-12, atol=0)
        single.close()
        multi[i].close()


def test_fill_multi_rejects_bad_arguments():
    h = pkg.Histogram([(10, 0.0, 1.0)])
    x = _t(np.zeros(10))
    with pytest.raises(pkg.BHistError):
        pkg.bh_fill_multi([h.h], [[3]], [False], 10, [x.data_ptr()])        # column out of range
    with pytest.raises(pkg.BHistError):
        pkg.bh_fill_multi([h.h], [[0]], [True], 10, [x.data_ptr()], None)   # weighted without w
    with pytest.raises(pkg.BHistError):
        pkg.bh_fill_multi([h.h, h.h], [[0], [0]], [False, False], 10, [x.data_ptr()])   # duplicate
    h.close()


@pytest.mark.parametrize("nbins,weighted", [(100, True), (100, False), (2000, True)])
def test_peaked_small_histograms_replicas(nbins, weighted):
    # Cauchy-peaked data on small bin spaces: PRIV with per-warp replicas and the
    # collision-adaptive weighted path (most lanes of a warp hit the same bin)
    rng = np.random.default_rng(nbins)
    n = 2_000_001
    x = 0.505 + 0.002 * np.tan(np.pi * (rng.random(n) - 0.5))
    w = rng.uniform(0.5, 1.5, n) if weighted else None
    axes = [(nbins, 0.0, 1.0)]
    ref = oracle.OracleHist(axes).fill([x], w).read()
    for s in (pkg.BH_STRATEGY_PRIV, pkg.BH_STRATEGY_CACHE, pkg.BH_STRATEGY_GLOBAL, pkg.BH_STRATEGY_SORT):
        compare(_gpu_fill(axes, [x], w, s), ref, weighted, f"peaked {nbins} strat {s}")


@pytest.mark.parametrize("nbins", [3, 9_999, 16_384, 16_385, 20_000])
@pytest.mark.parametrize("weighted", [False, True])
def test_variable_axis_guide_modes(nbins, weighted):
    # shared-memory guide tables: packed uint16 (n-1 < 16384, one load per event, cells
    # with >= 3 edges read the next entry) and plain uint16 above; edges with ties
    rng = np.random.default_rng(nbins)
    widths = rng.uniform(0.2, 1.8, nbins) ** 4          # very uneven widths: crowded cells
    edges = np.concatenate([[0.0], np.cumsum(widths)]) / widths.sum()
    edges[-1] = 1.0
    n = 1_000_003
    x = np.concatenate([rng.normal(0.5, 0.3, n - 4000), rng.choice(edges, 2000),
                        np.nextafter(rng.choice(edges, 2000), -np.inf)])
    w = rng.uniform(0.5, 1.5, n) if weighted else None
    ref = oracle.OracleHist([edges]).fill([x], w).read()
    compare(_gpu_fill([edges], [x], w), ref, weighted, f"guide modes n={nbins}")
    h = pkg.Histogram([edges])
    assert np.array_equal(h.find_bins([_t(x)]).cpu().numpy(), oracle.OracleHist([edges]).find_bins([x]))
    h.close()


@pytest.mark.parametrize("nb", [10, 50, 100])
def test_peaked_weighted_2d_warp_cache(nb):
    # weighted 2D fills of C5's peaked columns (Cauchy x, narrow Gaussian y): the
    # collision-adaptive sink with per-warp hot-bin caches (claims, evictions, drain)
    rng = np.random.default_rng(7 * nb)
    n = 3_000_017
    x = 0.505 + 0.002 * np.tan(np.pi * (rng.random(n) - 0.5))
    y = rng.normal(0.5, 0.05, n)
    w = rng.uniform(-0.5, 1.5, n)
    axes = [(nb, 0.0, 1.0), (nb, 0.0, 1.0)]
    ref = oracle.OracleHist(axes).fill([x, y], w).read()
    compare(_gpu_fill(axes, [x, y], w, pkg.BH_STRATEGY_PRIV, splits=2), ref, True, f"peaked 2D {nb}")


def test_bench_json_contract():
    """bench.py at N=1 on a reduced event count prints one JSON line with every key of
    the contract: roofline, e2e (incl. PCIe fraction), clocks, launches, CPU baselines."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, os.path.join(root, "bench.py"), "--steps", "3", "--warmup", "3", "--events", "4000000",
           "--e2e-steps", "1", "--secondary", "", "--cpu-sample", "200000"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks", "cpu_baseline"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 16 * 4_000_000 and e["d2h_bytes_per_step"] > 0
    assert 0 < e["pcie_frac"] < 1.5
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["config"]["workload"].startswith("C2")


def test_bench_two_ranks_exchange(tmp_path):
    """bench.py's N>1 path end to end on one GPU: 2 torchrun ranks (gloo backend so both
    may share cuda:0), contiguous shards, pack -> all-reduce -> unpack every step; the
    e2e leg asserts every rank ends with entries == N * world."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"), "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--backend", "gloo", "--events", "2000000", "--e2e-steps", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0 and d["scaling"] == "weak"
    assert d["cpu_baseline"] is None          # rank 0 at N=1 only


def test_fill_multi_fused_same_columns():
    # histograms over the same column(s) with different binnings share one fused pass
    # (k_fill_multi): fixed, variable (log) and 2D axes, unit and weighted
    rng = np.random.default_rng(21)
    n = 1_000_003
    x = rng.normal(0.5, 0.2, n)
    y = 0.505 + 0.002 * np.tan(np.pi * (rng.random(n) - 0.5))
    w = rng.uniform(0.5, 1.5, n)
    specs = [([(100, 0.0, 1.0)], [0], False), ([(37, -0.5, 1.5)], [0], False),
             ([np.geomspace(1e-3, 2.0, 301)], [0], False),
             ([(50, 0.0, 1.0)], [0], True), ([np.linspace(0.0, 1.0, 201)], [0], True),
             ([(20, 0.0, 1.0), (20, 0.4, 0.6)], [0, 1], True), ([(30, 0.0, 1.0), (30, 0.4, 0.6)], [0, 1], True)]
    cols = [_t(x), _t(y)]
    hs = [pkg.Histogram(ax) for ax, _, _ in specs]
    pkg.fill_multi(hs, [c for _, c, _ in specs], [wt for _, _, wt in specs], cols, _t(w))
    for h, (ax, c, wt) in zip(hs, specs):
        ref = oracle.OracleHist(ax).fill([[x, y][i] for i in c], w if wt else None).read()
        compare(h.read(), ref, wt, f"fused {ax}")
        h.close()


@pytest.mark.slow
def test_single_fill_above_2_31_events():
    """One bh_fill of 2^31 + 5 events (17 GB column): exercises the split into launches of
    <= 2^31 events and the 32-bit in-kernel indices; counts must equal the oracle's."""
    n = (1 << 31) + 5
    if torch.cuda.get_device_properties(0).total_memory < 40 * 2 ** 30:
        pytest.skip("needs > 40 GB of device memory")
    wl = bhgen.workload("C1", n)
    xd = torch.empty(n, dtype=torch.float64, device=DEV)
    chunk = 1 << 27
    host = torch.empty(chunk, dtype=torch.float64).pin_memory()
    for off in range(0, n, chunk):
        m = min(chunk, n - off)
        wl.column_ptr(0, off, m, host.data_ptr())
        xd[off:off + m].copy_(host[:m])
    h = pkg.Histogram([(100, 0.0, 1.0)])
    h.fill([xd])
    got = h.read()
    h.close()
    del xd
    ref = oracle_parallel("C1", n)
    compare(got, ref, False, "2^31+5")


# ------------------------------------------------------------------ fused Filter + Define (NEXT-1)
@pytest.mark.parametrize("strategy", [pkg.BH_STRATEGY_AUTO, pkg.BH_STRATEGY_GLOBAL, pkg.BH_STRATEGY_CACHE])
def test_fill_expr_filter_define(strategy):
    from oracle import expr
    rng = np.random.default_rng(5)
    n = 1_000_003
    x, y = rng.normal(0, 1, n), rng.normal(0, 1, n)
    w = rng.uniform(0.5, 1.5, n)
    x[::997] = np.nan
    P = pkg.Program(3)                     # r0 = x, r1 = y, r2 = w
    xx = P.mul(0, 0)
    yy = P.mul(1, 1)
    r = P.sqrt(P.add(xx, yy))              # Define("r", "sqrt(x*x+y*y)")
    cut = P.land(P.gt(0, P.const(-0.5)), P.lt(1, P.const(1.2)))   # Filter("x > -0.5 && y < 1.2")
    ww = P.mul(2, P.max(0, P.const(0.0)))  # weight = w * max(x, 0)
    cols = [_t(x), _t(y), _t(w)]
    for axes, regs, wreg in [([(100, 0.0, 3.0)], [r], -1), ([np.linspace(0, 3, 51) ** 1.5], [r], ww),
                             ([(40, 0.0, 3.0), (30, -1.0, 1.5)], [r, 1], 2)]:
        h = pkg.Histogram(axes, strategy=strategy)
        pkg.fill_expr(h, cols, P, regs, wreg, cut)
        ref = expr.fill_expr(axes, [x, y, w], P.ops, regs, wreg, cut).read()
        compare(h.read(), ref, wreg >= 0, f"expr {axes}")
        h.close()


def test_fill_expr_identity_equals_fill():
    wl = bhgen.workload("C2", 500_001)
    hist = wl.hists[0]
    cols, w = gen_columns(wl, hist, 0, wl.n_events)
    a = pkg.Histogram(oracle.oracle_axes(hist))
    a.fill([_t(cols[0])], _t(w))
    b = pkg.Histogram(oracle.oracle_axes(hist))
    pkg.fill_expr(b, [_t(cols[0]), _t(w)], pkg.Program(2), [0], 1, -1)
    ra, rb = a.read(), b.read()
    assert ra["entries"] == rb["entries"]
    np.testing.assert_allclose(ra["content"], rb["content"], rtol=1e-12, atol=0)
    a.close()
    b.close()


# ------------------------------------------------------------------ exact, deterministic weighted mode (NEXT-3)
@pytest.mark.parametrize("name", ["C2", "C3W", "C4W"])
def test_exact_mode_parity_and_reproducible(name):
    wl = bhgen.workload(name, 1_000_003)
    hist = wl.hists[0]
    axes = oracle.oracle_axes(hist)
    cols, w = gen_columns(wl, hist, 0, wl.n_events)
    ref = oracle.OracleHist(axes).fill(cols, w).read()
    a = _gpu_fill(axes, cols, w, pkg.BH_STRATEGY_EXACT)
    b = _gpu_fill(axes, cols, w, pkg.BH_STRATEGY_EXACT)
    compare(a, ref, True, f"exact {name}")
    assert np.array_equal(a["content"], b["content"]) and np.array_equal(a["sumw2"], b["sumw2"])
    assert np.array_equal(a["stats"], b["stats"])
    # the oracle's compensated sums are within ~1 ulp of exact: exact mode must be too
    nz = ref["content"] != 0
    rel = np.abs(a["content"][nz] - ref["content"][nz]) / np.abs(ref["content"][nz])
    assert rel.max() <= 4e-16


def test_exact_mode_is_correctly_rounded_sum():
    """Weights k * 2^-30 (k integer): the per-bin sums are then exact rationals we can form
    with Python integers; exact mode must return exactly their correctly rounded doubles,
    for sum(w) and for sum(RN(w*w))."""
    from fractions import Fraction
    rng = np.random.default_rng(77)
    n = 400_001
    x = rng.uniform(0, 1, n)
    k = rng.integers(2 ** 29, 3 * 2 ** 29, n)
    w = k.astype(np.float64) * 2.0 ** -30
    w[::5] *= -1.0
    axes = [(50, 0.0, 1.0)]
    got = _gpu_fill(axes, [x], w, pkg.BH_STRATEGY_EXACT)
    bins = oracle.OracleHist(axes).find_bins([x])
    ww = w * w
    for g in range(52):
        sel = bins == g
        s1 = sum((Fraction(float(v)) for v in w[sel]), Fraction(0))
        s2 = sum((Fraction(float(v)) for v in ww[sel]), Fraction(0))
        assert got["content"][g] == float(s1), g
        assert got["sumw2"][g] == float(s2), g


def test_exact_mode_nonfinite_weights_and_accumulation():
    rng = np.random.default_rng(3)
    n = 100_000
    x = rng.uniform(0, 1, n)
    w = rng.uniform(0.5, 1.5, n)
    w[17] = np.inf
    h = pkg.Histogram([(10, 0.0, 1.0)], strategy=pkg.BH_STRATEGY_EXACT)
    h.fill([_t(x)], _t(w))
    h.fill([_t(x)], _t(np.ones(n)))                    # second weighted fill accumulates
    r = h.read()
    b = int(x[17] * 10) + 1
    assert np.isinf(r["content"][b]) and np.isfinite(np.delete(r["content"], b)).all()
    ref = oracle.OracleHist([(10, 0.0, 1.0)]).fill([np.delete(x, 17)], np.delete(w, 17)).fill([x], np.ones(n)).read()
    other = np.arange(12) != b
    assert np.all(np.abs(r["content"][other] - ref["content"][other]) <= 1e-12 * ref["abs_content"][other])
    h.close()


# ------------------------------------------------------------------ float32 input columns (NEXT-2)
@pytest.mark.parametrize("name", ["C1", "C2", "C3W", "C4"])
@pytest.mark.parametrize("offset", [0, 1, 2, 3])
def test_fill_f32_equals_widened(name, offset):
    wl = bhgen.workload(name, 700_001)
    hist = wl.hists[0]
    axes = oracle.oracle_axes(hist)
    cols, w = gen_columns(wl, hist, 0, wl.n_events)
    cols32 = [c.astype(np.float32) for c in cols]
    w32 = None if w is None else w.astype(np.float32)
    ref = oracle.OracleHist(axes).fill([c.astype(np.float64) for c in cols32],
                                       None if w32 is None else w32.astype(np.float64)).read()
    h = pkg.Histogram(axes)
    tc = [torch.from_numpy(np.concatenate([np.zeros(offset, np.float32), c])).to(DEV)[offset:] for c in cols32]
    tw = None if w32 is None else torch.from_numpy(np.concatenate([np.zeros(offset, np.float32), w32])).to(DEV)[offset:]
    h.fill_f32(tc, tw)
    compare(h.read(), ref, w is not None, f"f32 {name} off {offset}")
    h.close()


def test_fill_f32_mixed_phases_and_tiny():
    rng = np.random.default_rng(9)
    for n in (0, 1, 3, 5, 17, 100_003):
        x = rng.uniform(-0.1, 1.1, n).astype(np.float32)
        y = rng.uniform(-0.1, 1.1, n + 1).astype(np.float32)[1:]       # different 16-byte phase
        axes = [(13, 0.0, 1.0), np.array([0.0, 0.2, 0.7, 1.0])]
        ref = oracle.OracleHist(axes).fill([x.astype(np.float64), y.astype(np.float64)]).read()
        h = pkg.Histogram(axes)
        if n:
            yt = torch.from_numpy(rng.uniform(0, 1, n + 1).astype(np.float32)).to(DEV)
            yt[1:] = torch.from_numpy(y).to(DEV)
            h.fill_f32([torch.from_numpy(x).to(DEV), yt[1:]])
        compare(h.read(), ref, False, f"f32 mixed n={n}")
        h.close()


# ------------------------------------------------------------------ SORT strategy (two-pass partitioned fill)
@pytest.mark.parametrize("name,n", [("C3", 1_000_003), ("C3W", 700_001), ("C4", 1_000_000), ("C4W", 600_007)])
@pytest.mark.parametrize("chunk", [4096, 65_537, 1 << 20])
def test_sort_many_chunks(name, n, chunk, monkeypatch):
    # chunks of 1 tile, of a ragged tile count and of many tiles: scratch reuse across
    # chunks, partial last tiles, partition totals re-zeroed by the plan kernel
    monkeypatch.setenv("BHIST_SORT_CHUNK", str(chunk))
    wl = bhgen.workload(name, n)
    hist = wl.hists[0]
    axes = oracle.oracle_axes(hist)
    cols, w = gen_columns(wl, hist, 0, n)
    ref = oracle.OracleHist(axes).fill(cols, w).read()
    got = _gpu_fill(axes, cols, w, pkg.BH_STRATEGY_SORT, splits=3)
    compare(got, ref, hist.weighted, f"{name} sort chunk={chunk}")


@pytest.mark.parametrize("shape,weighted", [((6000, 6000), False), ((4000, 4000), True), ((300, 300, 300), False),
                                            ((130, 1), True)])
def test_sort_many_partitions_and_ragged_last(shape, weighted):
    # up to ~2000 partitions (the SORT limit), a last partition shorter than 2^pb, variable
    # axes in pass 1, and a bin space smaller than one partition
    rng = np.random.default_rng(sum(shape))
    n = 1_500_017
    axes = []
    cols = []
    for k, nb in enumerate(shape):
        if k == 1:
            axes.append(np.cumsum(rng.uniform(0.5, 1.5, nb + 1)) / nb - 0.6)
        else:
            axes.append((nb, -0.1, 1.1))
        cols.append(rng.uniform(-0.2, 1.3, n))
    w = rng.uniform(-1.0, 2.0, n) if weighted else None
    ref = oracle.OracleHist(axes).fill(cols, w).read()
    compare(_gpu_fill(axes, cols, w, pkg.BH_STRATEGY_SORT), ref, weighted, f"sort {shape}")


@pytest.mark.parametrize("name,n", [("C3", 30_000_001), ("C3W", 6_000_007)])
def test_sort_pass2_spans_many_tile_batches(name, n):
    # a pass-2 CTA's stretch of (partition, tile) pairs exceeds one 2048-tile batch
    wl = bhgen.workload(name, n)
    hist = wl.hists[0]
    axes = oracle.oracle_axes(hist)
    cols, w = gen_columns(wl, hist, 0, n)
    ref = oracle.OracleHist(axes).fill(cols, w).read()
    compare(_gpu_fill(axes, cols, w, pkg.BH_STRATEGY_SORT), ref, hist.weighted, f"{name} sort n={n}")


@pytest.mark.parametrize("peaked", [False, True])
def test_auto_sort_probe(peaked):
    # AUTO + large unit-weight fills of a 1M-bin TH2D: the first fill runs CACHE and probes
    # a sample; later fills use SORT only for spread-out data.  Counts are exact either way.
    n = 40_000_000
    g = torch.Generator(device=DEV).manual_seed(5)
    def col():
        u = torch.rand(n, dtype=torch.float64, device=DEV, generator=g)
        return 0.505 + 0.002 * torch.tan(np.pi * (u - 0.5)) if peaked else u
    x, y = col(), col()                      # peaked: C4's Cauchy shape on both axes
    axes = [(1000, 0.0, 1.0), (1000, 0.0, 1.0)]
    h = pkg.Histogram(axes)
    ref = pkg.Histogram(axes, strategy=pkg.BH_STRATEGY_CACHE)
    assert h.strategy(False) == pkg.BH_STRATEGY_CACHE
    for _ in range(3):
        h.fill([x, y])
        ref.fill([x, y])
        torch.cuda.synchronize()
    assert h.strategy(False) == (pkg.BH_STRATEGY_CACHE if peaked else pkg.BH_STRATEGY_SORT)
    # the same probe decides weighted fills: GLOBAL (paired-lane REDs) unless a bin is hot
    assert h.strategy(True) == (pkg.BH_STRATEGY_CACHE if peaked else pkg.BH_STRATEGY_GLOBAL)
    a, b = h.read(), ref.read()
    assert a["entries"] == b["entries"] == 3 * n
    assert np.array_equal(a["content"], b["content"])
    assert a["stats"][0] == b["stats"][0]
    np.testing.assert_allclose(a["stats"], b["stats"], rtol=1e-12, atol=0)
    h.close()
    ref.close()


def test_strategy_resolution():
    h = pkg.Histogram([(1000, 0.0, 1.0), (1000, 0.0, 1.0)])
    assert h.strategy(False) == pkg.BH_STRATEGY_CACHE and h.strategy(True) == pkg.BH_STRATEGY_CACHE
    h.close()
    h = pkg.Histogram([(1000, 0.0, 1.0), (1000, 0.0, 1.0)], strategy=pkg.BH_STRATEGY_SORT)
    assert h.strategy(False) == pkg.BH_STRATEGY_SORT and h.strategy(True) == pkg.BH_STRATEGY_SORT
    h.close()
    # weighted partitions are 4x smaller: beyond 2048 of them SORT falls back to CACHE
    h = pkg.Histogram([(5000, 0.0, 1.0), (5000, 0.0, 1.0)], strategy=pkg.BH_STRATEGY_SORT)
    assert h.strategy(False) == pkg.BH_STRATEGY_SORT and h.strategy(True) == pkg.BH_STRATEGY_CACHE
    h.close()
    h = pkg.Histogram([(100, 0.0, 1.0)])
    assert h.strategy(False) == pkg.BH_STRATEGY_PRIV
    h.close()


# ------------------------------------------------------------------ int32 coordinate columns (NEXT-2)
@pytest.mark.parametrize("weighted", [False, True])
@pytest.mark.parametrize("offset", [0, 1, 3])
def test_fill_i32_equals_widened(weighted, offset):
    # integer coordinates (e.g. multiplicities) on fixed and variable axes, bins centred
    # on and between integers, flow on both sides; weights float32
    rng = np.random.default_rng(77 + offset)
    n = 1_000_003
    ax = [(20, -0.5, 19.5), np.array([-3.0, 0.0, 1.0, 2.0, 3.5, 7.0, 12.0, 40.0]), (7, 0.0, 14.0)]
    ci = [rng.poisson(6.0, n + offset).astype(np.int32) - 1, rng.integers(-5, 60, n + offset).astype(np.int32),
          rng.integers(-2, 20, n + offset).astype(np.int32)]
    wf = rng.uniform(-0.5, 1.5, n + offset).astype(np.float32) if weighted else None
    for dim in (1, 2, 3):
        axes = ax[:dim]
        cols = [c[offset:] for c in ci[:dim]]
        w = None if wf is None else wf[offset:]
        ref = oracle.OracleHist(axes).fill([c.astype(np.float64) for c in cols],
                                           None if w is None else w.astype(np.float64)).read()
        h = pkg.Histogram(axes)
        # slice on the device: columns start `offset` elements into their allocations
        h.fill_i32([torch.from_numpy(c).to(DEV)[offset:] for c in ci[:dim]],
                   None if wf is None else torch.from_numpy(wf).to(DEV)[offset:])
        compare(h.read(), ref, weighted, f"i32 dim={dim} offset={offset}")
        h.close()


def test_fill_i32_rejects_bad_arguments():
    h = pkg.Histogram([(10, 0.0, 10.0)])
    with pytest.raises(ValueError):
        h.fill_i32([torch.zeros(10, dtype=torch.int64, device=DEV)])
    with pytest.raises(pkg.BHistError):
        pkg.bh_fill_i32(h.h, 10, [None])
    h.close()
