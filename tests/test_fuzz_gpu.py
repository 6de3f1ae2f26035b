"""Randomized parity sweep: random histogram shapes (1-3 axes, fixed/variable, 1..~3000
bins), data mixes (uniform, normal, peaked, flow, NaN/inf, exact edges), weights
(none / positive / signed / zero), strategies, sizes, splits and misalignments — CUDA
path through the C ABI vs the oracle, with the north-star tolerances."""
import numpy as np
import pytest

import oracle
import paper_2401_13310_b200 as pkg
from _helpers import compare

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _axis(rng, max_bins):
    n = int(rng.integers(1, max_bins + 1))
    if rng.random() < 0.5:
        lo = float(rng.uniform(-50, 50))
        return (n, lo, lo + float(10 ** rng.uniform(-3, 3)))
    kind = rng.integers(3)
    if kind == 0:
        e = np.cumsum(rng.uniform(0.01, 1.0, n + 1))
    elif kind == 1:
        e = np.geomspace(1e-3, float(rng.uniform(1, 100)), n + 1)
    else:
        e = np.sort(rng.normal(0, 1, n + 1))
        e = e[np.concatenate([[True], np.diff(e) > 0])]
        if len(e) < 2:
            e = np.array([0.0, 1.0])
    return e


def _data(rng, ax, m):
    lo, hi = (ax[0], ax[-1]) if isinstance(ax, np.ndarray) else (ax[1], ax[2])
    span = hi - lo
    mode = rng.integers(4)
    if mode == 0:
        x = rng.uniform(lo - 0.1 * span, hi + 0.1 * span, m)
    elif mode == 1:
        x = rng.normal(lo + 0.5 * span, 0.3 * span, m)
    elif mode == 2:   # peaked
        x = lo + 0.5 * span + 1e-3 * span * np.tan(np.pi * (rng.random(m) - 0.5))
    else:             # exact edges and neighbours
        edges = ax if isinstance(ax, np.ndarray) else np.array([lo + i * span / ax[0] for i in range(ax[0] + 1)])
        x = edges[rng.integers(0, len(edges), m)]
        x = np.where(rng.random(m) < 0.5, x, np.nextafter(x, np.where(rng.random(m) < 0.5, -np.inf, np.inf)))
    k = max(1, m // 1000)
    idx = rng.integers(0, m, k) if m else []
    x[idx] = rng.choice([np.nan, np.inf, -np.inf, -0.0], k)
    return x


@pytest.mark.parametrize("seed", range(40))
def test_random_histograms(seed):
    rng = np.random.default_rng(1000 + seed)
    dim = int(rng.integers(1, 4))
    max_bins = {1: 3000, 2: 300, 3: 40}[dim]
    axes = [_axis(rng, max_bins) for _ in range(dim)]
    n = int(rng.choice([0, 1, 2, 7, 1000, 65_537, 300_001]))
    cols = [_data(rng, ax, n) for ax in axes]
    wmode = rng.integers(4)
    w = None if wmode == 0 else (rng.uniform(0.5, 1.5, n) if wmode == 1 else
                                 rng.normal(0, 1, n) if wmode == 2 else np.zeros(n))
    strategy = int(rng.choice([pkg.BH_STRATEGY_AUTO, pkg.BH_STRATEGY_GLOBAL, pkg.BH_STRATEGY_CACHE,
                                    pkg.BH_STRATEGY_SORT]))
    offset = int(rng.integers(0, 2))
    splits = int(rng.choice([1, 3]))
    ref = oracle.OracleHist(axes).fill(cols, w).read()
    h = pkg.Histogram(axes, strategy=strategy)
    tc = [torch.from_numpy(np.concatenate([np.zeros(offset), c])).to(DEV)[offset:] for c in cols]
    tw = None if w is None else torch.from_numpy(np.concatenate([np.zeros(offset), w])).to(DEV)[offset:]
    cuts = np.linspace(0, n, splits + 1).astype(int)
    for a, b in zip(cuts[:-1], cuts[1:]):
        h.fill([c[a:b] for c in tc], None if tw is None else tw[a:b])
    got = h.read()
    # bin indices are bit-exact
    if n:
        ob = oracle.OracleHist(axes).find_bins(cols)
        assert np.array_equal(h.find_bins(tc).cpu().numpy(), ob)
    h.close()
    if w is not None and wmode == 2:
        # signed weights: compare against sum|w| per bin (R14); stats likewise
        dc = np.abs(got["content"] - ref["content"])
        assert np.all(dc <= 1e-12 * ref["abs_content"] + 1e-300)
        assert got["entries"] == ref["entries"]
        assert np.all(np.abs(got["stats"] - ref["stats"]) <= 1e-12 * ref["stats_abs"] + 1e-300)
    else:
        compare(got, ref, w is not None, f"seed {seed}")
