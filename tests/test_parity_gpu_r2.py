"""GPU parity, round 2: per-event FindBin through every variable-axis search path, every
Filter+Define opcode, C5 at bench size, back-to-back host fills, and wrapper argument checks.
Bin indices bit-exact; weighted sums within 1e-12 of sum|term| (BASELINE.json north star)."""
import os

import numpy as np
import pytest

import bhgen
import oracle
import paper_2401_13310_b200 as pkg
from _helpers import compare, gen_columns, oracle_parallel

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _near(vals, k=3):
    """vals and +-1..k ulps around each."""
    out = [vals]
    up = dn = vals
    for _ in range(k):
        up, dn = np.nextafter(up, np.inf), np.nextafter(dn, -np.inf)
        out += [up, dn]
    return np.concatenate(out)


def _axes_under_test():
    wl = bhgen.workload("C2", 1000)
    c5 = bhgen.workload("C5", 1000)
    rng = np.random.default_rng(77)
    return {
        "C2 edges": wl.hists[0].axes[0].edges,                     # compact mode (8192 cells)
        "C5 H3 log": c5.hists[3].axes[0].edges,                     # crowded cells: packed guide
        "random 3000": np.cumsum(rng.uniform(1e-3, 1.0, 3001) ** 3) - 2.0,
        "uniform 16383": np.linspace(-1.0, 3.0, 16384),            # largest compact n
        "uniform 20000": np.linspace(0.0, 1.0, 20001),             # too many bins for compact
        "two bins": np.array([0.0, 0.25, 1.0]),
        "log 1e-3..2": np.geomspace(1e-3, 2.0, 1001),               # log-domain compact cells
        "log 1e-6..1e6 x 4000": np.geomspace(1e-6, 1e6, 4001),
    }


def _coords_for(edges, rng, m=200_000):
    lo, hi = edges[0], edges[-1]
    # random, every edge +-3 ulps, the guide-cell and quantized sub-cell (1/256) boundaries
    # +-2 ulps (where the compact search switches decisions), flow and special values
    sub = lo + (hi - lo) * (np.arange(0, 2 ** 15 * 256 + 1, 97) / (2 ** 15 * 256))
    xs = [rng.uniform(lo - 0.05 * (hi - lo), hi + 0.05 * (hi - lo), m), _near(edges), _near(sub, 2),
          np.array([np.nan, np.inf, -np.inf, -0.0, 0.0, 1e308, -1e308])]
    if lo > 0:   # log-domain cells: IEEE bit-pattern cell and sub-cell (1/256) boundaries +-2 ulps
        b0, bn = np.array([lo, hi]).view(np.int64)
        for sh in (34, 42):
            ks = np.arange(b0 >> sh, (bn >> sh) + 2, dtype=np.int64)
            xs.append(_near((ks << sh).view(np.float64), 2))
        xs.append(np.exp(rng.uniform(np.log(lo) - 0.1, np.log(hi) + 0.1, m // 2)))
    return np.concatenate(xs)


@pytest.mark.parametrize("compact", [True, False])
@pytest.mark.parametrize("search", ["staged", "global"])
def test_find_bins_every_search_path(compact, search, monkeypatch):
    """The per-event bin of the fills' own search (tables staged in shared memory: compact
    32-bit cells or float32 edges + guide) and of the float64 global search equals the
    oracle's binary search (reading R1) on random, edge, sub-cell-boundary and NaN/inf inputs."""
    if not compact:
        monkeypatch.setenv("BHIST_NO_COMPACT", "1")
    rng = np.random.default_rng(5 + compact)
    for name, edges in _axes_under_test().items():
        x = _coords_for(edges, rng)
        ref = oracle.OracleHist([edges]).find_bins([x])
        h = pkg.Histogram([edges])
        if search == "global":
            pkg.bh_set_debug(h.h, pkg.BH_DEBUG_FIND_BINS_GLOBAL)
        got = h.find_bins([_t(x)]).cpu().numpy()
        # the same events through a weighted fill (bins must match the per-event answer)
        w = rng.uniform(0.5, 1.5, len(x))
        h.fill([_t(x)], _t(w))
        compare(h.read(), oracle.OracleHist([edges]).fill([x], w).read(), True, name)
        h.close()
        bad = np.flatnonzero(got != ref)
        assert bad.size == 0, (name, compact, search, x[bad[:5]], got[bad[:5]], ref[bad[:5]])


def test_find_bins_mixed_axes_2d_3d():
    """2-D/3-D histograms mixing fixed and compact/packed variable axes (runtime per-axis
    dispatch in the staged search)."""
    rng = np.random.default_rng(9)
    ax = _axes_under_test()
    for axes in ([ax["C2 edges"], (100, 0.0, 1.0)], [(7, -1.0, 2.0), ax["C5 H3 log"], ax["two bins"]]):
        cols = []
        for a in axes:
            e = a if isinstance(a, np.ndarray) else np.linspace(a[1], a[2], a[0] + 1)
            c = _coords_for(e, rng, 100_000)
            cols.append(c)
        m = min(len(c) for c in cols)
        cols = [rng.permutation(c)[:m] for c in cols]
        ref = oracle.OracleHist(axes).find_bins(cols)
        h = pkg.Histogram(axes)
        got = h.find_bins([_t(c) for c in cols]).cpu().numpy()
        h.close()
        assert np.array_equal(got, ref), np.flatnonzero(got != ref)[:5]


# ------------------------------------------------------------------ Filter + Define: every opcode
def _expr_inputs(n, rng):
    a = rng.normal(0, 2, n)
    b = rng.normal(0.5, 1, n)
    c = rng.uniform(-3, 3, n)
    for arr in (a, b):
        arr[rng.integers(0, n, n // 50)] = np.nan
        arr[rng.integers(0, n, n // 200)] = np.inf
        arr[rng.integers(0, n, n // 200)] = -np.inf
        arr[rng.integers(0, n, n // 100)] = 0.0
        arr[rng.integers(0, n, n // 100)] = -0.0
    b[rng.integers(0, n, n // 20)] = a[rng.integers(0, n, n // 20)]        # equal operands for eq/ne/le/ge
    c[rng.integers(0, n, n // 10)] = 0.0                                  # select/logic on zero
    return a, b, c


@pytest.mark.parametrize("op", list(pkg.OPS))
def test_fill_expr_every_opcode(op):
    """Each of the 21 opcodes on the GPU against the numpy oracle (oracle/expr.py), its
    result used as the coordinate AND (for a second histogram) as the filter, so a wrong
    value or a wrong truth value both break parity.  Inputs carry NaN, +-inf, +-0."""
    from oracle import expr
    rng = np.random.default_rng(abs(hash(op)) % 2 ** 32)
    n = 300_001
    a, b, c = _expr_inputs(n, rng)
    prog = [(op, 3, 0, 1, 2, 1.25)]
    cols = [_t(a), _t(b), _t(c)]
    for axes, filt, wreg in (([(64, -6.0, 6.0)], -1, -1), ([(16, -3.0, 3.0)], 3, 2)):
        coord = 3 if filt < 0 else 2
        h = pkg.Histogram(axes)
        pkg.bh_fill_expr(h.h, n, [t.data_ptr() for t in cols], prog, [coord], wreg, filt,
                         torch.cuda.current_stream().cuda_stream)
        ref = expr.fill_expr(axes, [a, b, c], prog, [coord], wreg, filt).read()
        compare(h.read(), ref, wreg >= 0, f"{op} filter={filt}")
        h.close()


def test_fill_expr_long_program_all_registers():
    """A 32-op program touching all 16 registers (chained selects, divisions, sqrt of
    negatives) through a weighted 2-D fill."""
    from oracle import expr
    rng = np.random.default_rng(3)
    n = 200_003
    a, b, c = _expr_inputs(n, rng)
    names = list(pkg.OPS)
    prog = []
    for k in range(32):
        op = names[k % len(names)]
        dst = 3 + (k % 13)
        prog.append((op, dst, (k * 5) % 16, (k * 7 + 1) % 16, (k * 11 + 2) % 16, 0.5 + k))
    cols = [_t(a), _t(b), _t(c)]
    axes = [(20, -2.0, 2.0), (10, 0.0, 40.0)]
    h = pkg.Histogram(axes)
    pkg.bh_fill_expr(h.h, n, [t.data_ptr() for t in cols], prog, [15, 14], 2, 13,
                     torch.cuda.current_stream().cuda_stream)
    ref = expr.fill_expr(axes, [a, b, c], prog, [15, 14], 2, 13).read()
    compare(h.read(), ref, True, "32 ops")
    h.close()


# ------------------------------------------------------------------ C5 at the bench's size
@pytest.mark.slow
def test_c5_bench_size_against_sharded_oracle():
    """C5 as bench.py runs it at N=1 (1.25e8 device-resident events per GPU at 8 GPUs; the
    large-fill sinks the planner picks only at this size) against the oracle per histogram,
    through both plans of bh_fill_multi (per-histogram passes, the one-pass kernel)."""
    n = 125_000_000
    wl = bhgen.workload("C5", n)
    cols = [_t(wl.column(c, 0, n)) for c in range(len(wl.columns))]
    w = _t(wl.column(wl.wcol, 0, n))
    got = {}
    for mode in (pkg.BH_MULTI_PASSES, pkg.BH_MULTI_ONE_PASS):     # both plans of bh_fill_multi
        hs = [pkg.Histogram(oracle.oracle_axes(hist)) for hist in wl.hists]
        if mode == pkg.BH_MULTI_ONE_PASS:
            pkg.bh_set_debug(hs[0].h, pkg.BH_DEBUG_REQUIRE_JIT)
        pkg.fill_multi(hs, [hist.cols for hist in wl.hists], [hist.weighted for hist in wl.hists], cols, w, mode=mode)
        got[mode] = [h.read() for h in hs]
        for h in hs:
            h.close()
    del cols, w
    torch.cuda.empty_cache()
    for i, hist in enumerate(wl.hists):
        ref = oracle_parallel("C5", n, hidx=i)
        for mode, g in got.items():
            compare(g[i], ref, hist.weighted, f"C5 H{i} plan {mode}")


# ------------------------------------------------------------------ host -> device path
def test_fill_host_back_to_back_calls_while_stream_busy():
    """bh_fill_host returns once the HOST bytes are consumed; its fills may
    still be queued.  A second call made at once must not overwrite a staging slot those
    queued fills still read: keep the stream busy, fill twice, compare."""
    rng = np.random.default_rng(12)
    axes = [(1000, 0.0, 1.0)]
    n = 1 << 16
    x1, x2 = rng.uniform(0, 0.5, n), rng.uniform(0.5, 1.0, n)
    h = pkg.Histogram(axes)
    pkg.bh_set_chunk(h.h, 1 << 14)                       # 4 chunks per call through 2 slots
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        torch.cuda._sleep(200_000_000)                   # ~0.1 s of GPU time queued on s
        h.fill_host([x1], stream=s)
        h.fill_host([x2], stream=s)
    s.synchronize()
    ref = oracle.OracleHist(axes).fill([x1]).fill([x2]).read()
    compare(h.read(), ref, False, "back-to-back fill_host")
    h.close()


def test_wrapper_rejects_wrong_columns():
    """dtype / length / contiguity / device checks before any pointer
    reaches the C ABI."""
    h = pkg.Histogram([(10, 0.0, 1.0)])
    with pytest.raises(ValueError):
        h.fill_host([np.zeros(10, dtype=np.float32)])
    with pytest.raises(ValueError):
        h.fill_host([np.zeros(10)], w=np.zeros(9))
    with pytest.raises(ValueError):
        h.fill_host([np.zeros(20)[::2]])
    with pytest.raises(ValueError):
        h.fill_host([torch.zeros(10, device=DEV)])
    with pytest.raises(ValueError):
        h.fill([torch.zeros(10, device=DEV, dtype=torch.float32)])
    with pytest.raises(ValueError):
        h.fill([torch.zeros(10, device=DEV)], torch.zeros(9, device=DEV, dtype=torch.float64))
    with pytest.raises(ValueError):
        h.fill([torch.zeros(10, dtype=torch.float64)])          # host tensor to a device fill
    with pytest.raises(ValueError):
        h.fill([torch.zeros(10, device=DEV, dtype=torch.float64), torch.zeros(10, device=DEV, dtype=torch.float64)])
    if torch.cuda.device_count() > 1:
        with pytest.raises(ValueError):
            h.fill([torch.zeros(10, device="cuda:1", dtype=torch.float64)])
    h.close()


def test_forced_priv_weighted_falls_back_when_cells_do_not_fit():
    """PRIV is accepted for a bin space whose unit-weight counters fit but
    whose 16-byte weighted cells do not; weighted fills then take CACHE and stay correct."""
    axes = [(150, 0.0, 1.0), (150, 0.0, 1.0)]        # 23,104 bins: 92 KB unit, 370 KB weighted
    h = pkg.Histogram(axes, strategy=pkg.BH_STRATEGY_PRIV)
    assert h.strategy(False) == pkg.BH_STRATEGY_PRIV and h.strategy(True) == pkg.BH_STRATEGY_CACHE
    rng = np.random.default_rng(4)
    x, y, w = rng.uniform(0, 1, 500_000), rng.normal(0.5, 0.2, 500_000), rng.uniform(0.5, 1.5, 500_000)
    h.fill([_t(x), _t(y)], _t(w))
    compare(h.read(), oracle.OracleHist(axes).fill([x, y], w).read(), True, "forced PRIV weighted")
    h.close()


# ------------------------------------------------------------------ host float32 / int32 columns (NEXT-2)
@pytest.mark.parametrize("kind", ["f32", "i32"])
@pytest.mark.parametrize("weighted", [False, True])
def test_fill_host_4byte_columns(kind, weighted):
    """bh_fill_host_f32 / _i32: host 4-byte columns through the staging ring (chunks of
    2x the float64 chunk), equal to the oracle on the exactly widened columns."""
    rng = np.random.default_rng(31)
    n = 1_000_003
    if kind == "f32":
        x = rng.normal(0.5, 0.2, n).astype(np.float32)
        y = rng.uniform(-0.1, 1.1, n).astype(np.float32)
        axes = [bhgen.workload("C2", 10).hists[0].axes[0].edges, (50, 0.0, 1.0)]
    else:
        x = rng.integers(-5, 120, n).astype(np.int32)
        y = rng.poisson(7.0, n).astype(np.int32)
        axes = [(100, 0.0, 100.0), np.array([0.0, 2.0, 5.0, 6.0, 7.0, 8.0, 12.0, 30.0])]
    w = rng.uniform(0.5, 1.5, n).astype(np.float32) if weighted else None
    h = pkg.Histogram(axes)
    pkg.bh_set_chunk(h.h, 100_000)
    xs = [torch.from_numpy(x).pin_memory(), torch.from_numpy(y)]       # pinned and pageable
    tw = None if w is None else torch.from_numpy(w).pin_memory()
    (h.fill_host_f32 if kind == "f32" else h.fill_host_i32)(xs, tw)
    ref = oracle.OracleHist(axes).fill([x.astype(np.float64), y.astype(np.float64)],
                                       None if w is None else w.astype(np.float64)).read()
    compare(h.read(), ref, weighted, f"fill_host_{kind}")
    h.close()


# ------------------------------------------------------------------ multi-histogram exchange
def test_pack_multi_layout_and_roundtrip():
    """bh_pack_multi: histograms back to back, unit ones without sumw2; unpack restores
    every state (unit: sumw2 := content); a unit entry for a weighted histogram is refused."""
    wl = bhgen.workload("C5", 300_001)
    n = wl.n_events
    cols = [_t(wl.column(c, 0, n)) for c in range(len(wl.columns))]
    w = _t(wl.column(wl.wcol, 0, n))
    hs = [pkg.Histogram(oracle.oracle_axes(hist)) for hist in wl.hists]
    pkg.fill_multi(hs, [hist.cols for hist in wl.hists], [hist.weighted for hist in wl.hists], cols, w)
    before = [h.read() for h in hs]
    unit = [not hist.weighted for hist in wl.hists]
    handles = [h.h for h in hs]
    size = pkg.bh_packed_size_multi(handles, unit)
    assert size == sum((1 if u else 2) * h.nbins_total + h.nstats + 1 for h, u in zip(hs, unit))
    buf = torch.empty(size, dtype=torch.float64, device=DEV)
    pkg.bh_pack_multi(handles, unit, buf.data_ptr(), torch.cuda.current_stream().cuda_stream)
    b = buf.cpu().numpy()
    off = 0
    for r, u, h in zip(before, unit, hs):
        assert np.array_equal(b[off:off + h.nbins_total], r["content"])
        off += h.nbins_total
        if not u:
            assert np.array_equal(b[off:off + h.nbins_total], r["sumw2"])
            off += h.nbins_total
        assert np.array_equal(b[off:off + h.nstats], r["stats"])
        off += h.nstats
        assert b[off] == r["entries"]
        off += 1
    for h in hs:
        h.reset()
    pkg.bh_unpack_multi(handles, unit, buf.data_ptr(), torch.cuda.current_stream().cuda_stream)
    for h, r, u in zip(hs, before, unit):
        a = h.read()
        for k in ("content", "sumw2", "stats"):
            assert np.array_equal(a[k], r[k]), k
        assert a["entries"] == r["entries"]
        if u:   # a reduced unit-weight state still reads as TH1I counts (reading R18)
            i32 = h.read(content_type=pkg.BH_CONTENT_I32)
            assert np.array_equal(i32["content"], r["content"].astype(np.int64))
    with pytest.raises(pkg.BHistError):       # histogram 1 is weighted: no unit packing
        hs[1].fill([cols[1]], w)
        pkg.bh_pack_multi(handles, [True] * len(hs), buf.data_ptr(), torch.cuda.current_stream().cuda_stream)
    for h in hs:
        h.close()


def _free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _bench_ranks(tmp_path, world, backend, config, events, exchange):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    dump = str(tmp_path / f"dump_{config}_{exchange}.npz")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"),
           "--gpus", str(world), "--steps", "3", "--warmup", "3", "--backend", backend, "--events", str(events),
           "--e2e-steps", "1", "--config", config, "--exchange", exchange, "--dump", dump]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    return json.loads(lines[0]), np.load(dump)


@pytest.mark.parametrize("config,exchange", [("C2", "reduce"), ("C5", "allreduce"), ("C3", "reduce")])
def test_bench_two_ranks_reduced_state_matches_oracle(tmp_path, config, exchange):
    """bench.py --gpus 2 (two gloo ranks sharing cuda:0): each rank fills its contiguous
    shard [r N, (r+1) N), one collective per step sums all histograms; the state rank 0
    ends with equals the oracle over all 2N events."""
    events = 400_003
    d, z = _bench_ranks(tmp_path, 2, "gloo", config, events, exchange)
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "weak"
    wl = bhgen.workload(config, 2 * events)
    for i, hist in enumerate(wl.hists):
        ref = oracle_parallel(config, 2 * events, hidx=i, nproc=4)
        got = {"content": z[f"content{i}"], "sumw2": z[f"sumw2{i}"], "stats": z[f"stats{i}"],
               "entries": int(z[f"entries{i}"])}
        compare(got, ref, hist.weighted, f"{config} H{i} {exchange}")


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("exchange", ["reduce", "allreduce"])
def test_nccl_two_gpus_reduced_state_matches_oracle(tmp_path, exchange):
    """The same over NCCL on two GPUs (skipped on one-GPU boxes)."""
    events = 2_000_003
    d, z = _bench_ranks(tmp_path, 2, "nccl", "C5", events, exchange)
    wl = bhgen.workload("C5", 2 * events)
    for i, hist in enumerate(wl.hists):
        ref = oracle_parallel("C5", 2 * events, hidx=i)
        got = {"content": z[f"content{i}"], "sumw2": z[f"sumw2{i}"], "stats": z[f"stats{i}"],
               "entries": int(z[f"entries{i}"])}
        compare(got, ref, hist.weighted, f"nccl C5 H{i}")


# ------------------------------------------------------------------ one-pass fused multi-histogram fill (JIT)
def _fused_case(name, rng, n):
    """(columns, w, [(axes, col indices, weighted)]) of a histogram set."""
    if name == "C5":
        wl = bhgen.workload("C5", n)
        cols = [wl.column(c, 0, n) for c in range(len(wl.columns))]
        return cols, wl.column(wl.wcol, 0, n), [(oracle.oracle_axes(h), h.cols, h.weighted) for h in wl.hists]
    x = rng.normal(0.5, 0.2, n)
    y = 0.505 + 0.002 * np.tan(np.pi * (rng.random(n) - 0.5))      # Cauchy-peaked
    z = rng.uniform(-0.1, 1.1, n)
    w = rng.uniform(-0.5, 1.5, n)
    c2 = bhgen.workload("C2", 10).hists[0].axes[0].edges
    if name == "3d+global":
        specs = [([(100, 0.0, 1.0)] * 3, [0, 1, 2], False),            # 1M bins: L2 sink
                 ([(150, 0.0, 1.0), (150, 0.0, 1.0)], [2, 0], True),   # 22,801 weighted cells: L2 sink
                 ([c2], [0], True), ([(20, 0.4, 0.6), (30, 0.0, 1.0)], [1, 2], True),
                 ([np.geomspace(1e-3, 2.0, 801)], [2], False)]
    elif name == "small":
        specs = [([(10, 0.0, 1.0)], [0], False), ([(7, 0.45, 0.55)], [1], True), ([np.array([0.0, 0.3, 0.31, 1.0])], [2], True)]
    else:
        raise KeyError(name)
    return [x, y, z], w, specs


@pytest.mark.parametrize("name,n", [("C5", 2_000_003), ("3d+global", 1_000_001), ("small", 300_007), ("small", 5),
                                    ("C5", 33)])
def test_fused_one_pass_against_oracle(name, n):
    """bh_fill_multi's run-time specialized one-pass kernel (BH_DEBUG_REQUIRE_JIT: no fallback):
    one launch for the whole set, every histogram equal to its own oracle fill."""
    rng = np.random.default_rng(n)
    cols, w, specs = _fused_case(name, rng, n)
    hs = [pkg.Histogram(ax) for ax, _, _ in specs]
    pkg.bh_set_debug(hs[0].h, pkg.BH_DEBUG_REQUIRE_JIT)
    tc = [_t(c) for c in cols]
    tw = _t(w)
    l0 = pkg.bh_launch_count(hs[0].h)
    for rep in range(2):                      # accumulation across fills (include-initial)
        pkg.fill_multi(hs, [c for _, c, _ in specs], [wt for _, _, wt in specs], tc, tw)
    assert pkg.bh_launch_count(hs[0].h) - l0 == 2
    for h, (ax, c, wt) in zip(hs, specs):
        o = oracle.OracleHist(ax)
        for rep in range(2):
            o.fill([cols[i] for i in c], w if wt else None)
        compare(h.read(), o.read(), wt, f"{name} {ax if not isinstance(ax[0], np.ndarray) else 'var'}")
        h.close()


# ------------------------------------------------------------------ AUTO's SORT decision (device-side, data-only)
@pytest.mark.slow
def test_auto_sort_decision_is_deterministic_and_matches_oracle():
    """AUTO decides SORT vs CACHE on the device from a sample of the first large unit-weight
    fill (both paths launched, gated): two fresh histograms fed the same fills end bitwise
    identical (the choice never depends on host timing), the spread-out C3 shape picks
    SORT, and the result equals the oracle; bh_reset re-decides."""
    n = 40_000_001
    wl = bhgen.workload("C3", n)
    cols = [wl.column(c, 0, n) for c in wl.hists[0].cols]
    tc = [_t(c) for c in cols]
    axes = oracle.oracle_axes(wl.hists[0])
    runs = []
    for rep in range(2):
        h = pkg.Histogram(axes)
        h.fill(tc)
        h.fill(tc)
        runs.append((h.read(), h.strategy(False)))
        h.reset()
        h.fill(tc)
        assert h.read()["entries"] == n
        h.close()
    (a, sa), (b, sb) = runs
    assert sa == sb == pkg.BH_STRATEGY_SORT
    assert np.array_equal(a["content"], b["content"]) and a["stats"].tobytes() == b["stats"].tobytes()
    ref = oracle_parallel("C3", n)
    ref2 = {k: (2 * v if k != "entries" else 2 * v) for k, v in ref.items()}
    compare(a, ref2, False, "AUTO->SORT x2")


# ------------------------------------------------------------------ AUTO's weighted GLOBAL/CACHE decision
@pytest.mark.slow
@pytest.mark.parametrize("name,want", [("C3W", "global"), ("C4W", "cache")])
def test_auto_weighted_global_decision_matches_oracle(name, want):
    """Weighted fills of a bin space that does not fit PRIV: the device probe picks GLOBAL
    (paired-lane L2 REDs) on spread-out data and CACHE on a hot bin (C4w: ~43% of the events
    in one cell), both launched gated; two fresh histograms end bitwise identical in counts
    and stats, and the result equals the oracle within 1e-12 of sum|term|."""
    n = 40_000_003
    wl = bhgen.workload(name, n)
    hist = wl.hists[0]
    tc = [_t(wl.column(c, 0, n)) for c in hist.cols]
    tw = _t(wl.column(wl.wcol, 0, n))
    axes = oracle.oracle_axes(hist)
    runs = []
    for rep in range(2):
        h = pkg.Histogram(axes)
        h.fill(tc, tw)
        runs.append((h.read(), h.strategy(True)))
        h.close()
    (a, sa), (b, sb) = runs
    strat = {"global": pkg.BH_STRATEGY_GLOBAL, "cache": pkg.BH_STRATEGY_CACHE}[want]
    assert sa == sb == strat
    assert a["entries"] == b["entries"] == n
    compare(a, oracle_parallel(name, n), True, f"AUTO weighted {name} -> {want}")


# ------------------------------------------------------------------ TH1F / TH1I contents (reading R18)
@pytest.mark.parametrize("name,weighted", [("C1", False), ("C2", True), ("C3", False)])
def test_read_as_float32_and_int32_contents(name, weighted):
    """bh_read_as narrows the exact device state once: float32 = RN_f32(float64 content),
    int32 = the unit-weight count (TH1I), against the oracle's float64 contents."""
    n = 1_000_003
    wl = bhgen.workload(name, n)
    hist = wl.hists[0]
    h = pkg.Histogram(oracle.oracle_axes(hist))
    h.fill([_t(wl.column(c, 0, n)) for c in hist.cols], _t(wl.column(wl.wcol, 0, n)) if weighted else None)
    d = h.read()
    f = h.read(content_type=pkg.BH_CONTENT_F32)
    assert f["content"].dtype == np.float32 and f["sumw2"].dtype == np.float32
    assert np.array_equal(f["content"], d["content"].astype(np.float32))      # the definition, bin by bin
    assert np.array_equal(f["sumw2"], d["sumw2"].astype(np.float32))
    assert f["entries"] == n and np.array_equal(f["stats"], d["stats"])
    ref = oracle_parallel(name, n)
    rf = ref["content"].astype(np.float32)
    # float64 results agree within 1e-12 relative; their float32 roundings within one float32 ulp
    assert np.all(np.abs(f["content"] - rf) <= np.spacing(np.abs(rf)))
    if weighted:
        with pytest.raises(pkg.BHistError):
            h.read(content_type=pkg.BH_CONTENT_I32)
    else:
        i = h.read(content_type=pkg.BH_CONTENT_I32)
        assert i["content"].dtype == np.int32
        assert np.array_equal(i["content"], ref["content"].astype(np.int64))
        assert np.array_equal(i["sumw2"], i["content"])
    h.close()


def test_read_as_int32_saturates():
    """A TH1I bin saturates at INT32_MAX (ROOT's TH1I); the float32 content is RN_f32 of the
    exact count: 9 fills of 2^28 events into one bin = 2415919104 > 2^31 - 1."""
    m = 1 << 28
    x = torch.full((m,), 0.5, dtype=torch.float64, device=DEV)
    h = pkg.Histogram([(1, 0.0, 1.0)])
    for _ in range(9):
        h.fill([x])
    i = h.read(content_type=pkg.BH_CONTENT_I32)
    f = h.read(content_type=pkg.BH_CONTENT_F32)
    assert i["content"].tolist() == [0, 2147483647, 0] and i["entries"] == 9 * m
    assert f["content"].tolist() == [0.0, 2415919104.0, 0.0]
    h.close()


# ------------------------------------------------------------------ hot-cell window (weighted PRIVA)
@pytest.mark.parametrize("hidx,n", [(7, 1 << 23), (7, (1 << 22) + 7), (5, 1 << 23), (1, 1 << 23)])
def test_hot_window_weighted_priva_matches_oracle(hidx, n):
    """C5's peaked weighted H7 (50x50, ~75% of the events in 8 cells) takes the lane-private
    window (device probe, gated kernels); H5/H1 (spread out) take plain PRIVA.  Both equal the
    oracle; a second fill and a reset re-probe keep the result exact."""
    wl = bhgen.workload("C5", n)
    hist = wl.hists[hidx]
    cols = [_t(wl.column(c, 0, n)) for c in hist.cols]
    w = _t(wl.column(wl.wcol, 0, n))
    h = pkg.Histogram(oracle.oracle_axes(hist))
    h.fill(cols, w)
    h.fill(cols, w)
    got = h.read()
    ref = oracle_parallel("C5", n, hidx=hidx)
    compare(got, {k: 2 * v for k, v in ref.items()}, True, f"C5 H{hidx} x2 (hot window)")
    h.reset()
    h.fill(cols, w)
    compare(h.read(), ref, True, f"C5 H{hidx} after reset")
    h.close()


# ------------------------------------------------------------------ unit-weight WINDOW (AUTO probe decision 2)
@pytest.mark.slow
@pytest.mark.parametrize("case", ["C5 H6", "1D 200k gauss"])
def test_auto_window_unit_matches_oracle(case):
    """Large unit-weight bin spaces whose events concentrate in a box (C5's H6: 1000x1000 on
    two Gaussians; a 200,000-bin 1-D Gaussian) take CACHE with the probe's dense box of
    private shared-memory counts: counts bit-exact vs the oracle, fresh histograms identical."""
    n = 40_000_001
    if case == "C5 H6":
        wl = bhgen.workload("C5", n)
        hist = wl.hists[6]
        cols = [wl.column(c, 0, n) for c in hist.cols]
        axes = oracle.oracle_axes(hist)
        ref = oracle_parallel("C5", n, hidx=6)
    else:
        wl = bhgen.workload("C2", n)                  # N(0.5, 0.15) column
        cols = [wl.column(wl.hists[0].cols[0], 0, n)]
        axes = [(200_000, 0.0, 1.0)]
        ref = oracle.OracleHist(axes).fill(cols).read()
    tc = [_t(c) for c in cols]
    outs = []
    for rep in range(2):
        h = pkg.Histogram(axes)
        h.fill(tc)
        h.fill(tc)
        outs.append(h.read())
        h.close()
    a, b = outs
    assert np.array_equal(a["content"], b["content"]) and a["stats"].tobytes() == b["stats"].tobytes()
    compare(a, {k: 2 * v for k, v in ref.items()}, False, f"AUTO window {case}")


# ------------------------------------------------------------------ every AUTO-gated kernel on small inputs
@pytest.mark.parametrize("name,hidx", [("C3", 0), ("C3W", 0), ("C4", 0), ("C4W", 0), ("C5", 6), ("C5", 7),
                                       ("C5", 5), ("C5", 1)])
@pytest.mark.parametrize("n", [40_009, 100_003])
def test_auto_probe_paths_small_inputs(name, hidx, n, monkeypatch):
    """With BHIST_AUTO_MIN_EVENTS=1 the device probes and their gated kernels (SORT, GLOBAL
    paired REDs, the unit WINDOW box, CACHE / PRIVA + lane window) run on small, ragged fills;
    two fills plus a misaligned third equal the oracle (counts exact, sums within 1e-12)."""
    monkeypatch.setenv("BHIST_AUTO_MIN_EVENTS", "1")
    wl = bhgen.workload(name, n)
    hist = wl.hists[hidx]
    cols = [wl.column(c, 0, n) for c in hist.cols]
    w = wl.column(wl.wcol, 0, n) if hist.weighted else None
    h = pkg.Histogram(oracle.oracle_axes(hist))
    tc = [_t(c) for c in cols]
    tw = _t(w) if w is not None else None
    h.fill(tc, tw)
    h.fill(tc, tw)
    h.fill([c[1:] for c in tc], tw[1:] if tw is not None else None)      # peeled / misaligned path
    ref = oracle.OracleHist(oracle.oracle_axes(hist))
    ref.fill(cols, w).fill(cols, w).fill([c[1:] for c in cols], w[1:] if w is not None else None)
    compare(h.read(), ref.read(), hist.weighted, f"{name} H{hidx} n={n}")
    h.close()


@pytest.mark.slow
def test_auto_decision_then_smaller_fills_with_fewer_candidates():
    """The probes decide once (first large fill); a later, smaller fill that launches fewer
    candidate kernels (C3w: GLOBAL needs >= 39M events, the hot-cell probe only 4M) still
    runs exactly one sink: the plain kernel takes every word whose kernel is not launched."""
    n1, n2 = 40_000_003, 5_000_011
    wl = bhgen.workload("C3W", n1)
    hist = wl.hists[0]
    cols = [wl.column(c, 0, n1) for c in hist.cols]
    w = wl.column(wl.wcol, 0, n1)
    tc, tw = [_t(c) for c in cols], _t(w)
    h = pkg.Histogram(oracle.oracle_axes(hist))
    h.fill(tc, tw)                                   # probes: GLOBAL
    assert h.strategy(True) == pkg.BH_STRATEGY_GLOBAL
    h.fill([c[:n2] for c in tc], tw[:n2])            # no GLOBAL candidate: CACHE must run
    ref = oracle.OracleHist(oracle.oracle_axes(hist))
    ref.fill(cols, w).fill([c[:n2] for c in cols], w[:n2])
    compare(h.read(), ref.read(), True, "C3w 40M then 5M")
    h.close()


@pytest.mark.slow
def test_auto_decision_after_reset_follows_the_inputs():
    """bh_reset keeps AUTO's device decision for fills over the same input buffers (the bench's
    repeated steps) and makes it again for other buffers: a histogram that chose SORT on
    uniform data chooses CACHE after a reset and a fill of peaked data; counts stay exact."""
    n = 40_000_000
    g = torch.Generator(device=DEV).manual_seed(11)
    u = [torch.rand(n, dtype=torch.float64, device=DEV, generator=g) for _ in range(2)]
    pk = [0.505 + 0.002 * torch.tan(np.pi * (torch.rand(n, dtype=torch.float64, device=DEV, generator=g) - 0.5))
          for _ in range(2)]
    axes = [(1000, 0.0, 1.0), (1000, 0.0, 1.0)]
    h = pkg.Histogram(axes)
    ref = pkg.Histogram(axes, strategy=pkg.BH_STRATEGY_CACHE)
    h.fill(u)
    assert h.strategy(False) == pkg.BH_STRATEGY_SORT
    h.reset()
    h.fill(u)                                       # same buffers: decision kept
    assert h.strategy(False) == pkg.BH_STRATEGY_SORT
    ref.fill(u)
    assert np.array_equal(h.read()["content"], ref.read()["content"])
    h.reset()
    ref.reset()
    h.fill(pk)                                      # other buffers: decided again
    ref.fill(pk)
    assert h.strategy(False) == pkg.BH_STRATEGY_CACHE
    a, b = h.read(), ref.read()
    assert np.array_equal(a["content"], b["content"]) and a["entries"] == b["entries"] == n
    h.close()
    ref.close()
