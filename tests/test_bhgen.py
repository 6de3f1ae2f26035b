"""The shared input generator: determinism, chunk invariance, known SplitMix64 values."""
import numpy as np

import bhgen


def test_splitmix64_reference_values():
    # SplitMix64 (Steele, Lea, Flood 2014) first outputs from state 0: the state is advanced by
    # the golden gamma before mixing, so splitmix64(0) = 0xe220a8397b1dcdaf.
    L = bhgen.lib()
    assert L.bg_splitmix64(0) == 0xE220A8397B1DCDAF
    assert L.bg_splitmix64(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4


def test_u01_mapping_range_and_determinism():
    x = bhgen.sample(bhgen.UNIFORM, 42, 0, 100000, 0.0, 1.0)
    assert x.min() >= 0.0 and x.max() < 1.0
    assert np.all(x * 2.0 ** 53 == np.floor(x * 2.0 ** 53))   # 53-bit mantissa mapping (SPEC D15)
    assert np.array_equal(x, bhgen.sample(bhgen.UNIFORM, 42, 0, 100000, 0.0, 1.0))
    assert abs(x.mean() - 0.5) < 0.002


def test_chunk_invariance_all_kinds():
    for kind, p0, p1 in [(bhgen.UNIFORM, 0.5, 1.5), (bhgen.GAUSS, 0.5, 0.15), (bhgen.CAUCHY, 0.505, 0.002),
                         (bhgen.EXP, 5.0, 0.0)]:
        full = bhgen.sample(kind, 7, 0, 300001, p0, p1, nthreads=4)
        parts = np.concatenate([bhgen.sample(kind, 7, a, b - a, p0, p1, nthreads=1)
                                for a, b in [(0, 1), (1, 99999), (99999, 300001)]])
        assert np.array_equal(full, parts)


def test_edges_strictly_increasing_and_exact_ends():
    e = bhgen.c2_edges()
    assert len(e) == 10001 and e[0] == 0.0 and e[-1] == 1.0 and np.all(np.diff(e) > 0)
    d = np.diff(e)
    assert d.max() / d.min() < 3.0001
    lg = bhgen.edges_log(1e-3, 2.0, 1000)
    assert lg[0] == 1e-3 and lg[-1] == 2.0 and np.all(np.diff(lg) > 0)


def test_workloads_defined():
    for name in ("C1", "C2", "C3", "C3W", "C4", "C4W", "C5"):
        wl = bhgen.workload(name, 1000)
        assert wl.n_events == 1000 and wl.hists
        for h in wl.hists:
            for c in h.cols:
                assert 0 <= c < len(wl.columns)
    assert bhgen.workload("C2").bytes_per_event == 16
    assert bhgen.workload("C5").bytes_per_event == 56
    assert bhgen.shard(10, 0, 3) == (0, 3) and bhgen.shard(10, 2, 3) == (6, 10)
