"""Pins for the CPU oracle (oracle/bhist_oracle.c) against things other than itself:
worked examples printed in SPEC.md (tests/golden/spec_examples.json), hand-derived
IEEE cases (tests/golden/ieee_pins.json), exact rational arithmetic (fractions),
brute-force linear scans, closed-form moments of the input laws (scipy quadrature),
and invariants (conservation, bijection, bulk-split / merge invariance).
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import bhgen
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _x(v):
    if isinstance(v, str):
        return float(v) if v in ("nan", "inf", "-inf") else float.fromhex(v)
    return float(v)


# ------------------------------------------------------------------ SPEC worked examples
def test_spec_find_bin_fixed():
    for ex in _load("spec_examples.json")["find_bin_fixed"]:
        assert oracle.find_bin_fixed(ex["nbins"], ex["xmin"], ex["xmax"], ex["x"]) == ex["bin"], ex["cite"]


def test_spec_find_bin_variable():
    for ex in _load("spec_examples.json")["find_bin_variable"]:
        assert oracle.find_bin_variable(ex["edges"], ex["x"]) == ex["bin"], ex["cite"]


def test_spec_global_bin():
    for ex in _load("spec_examples.json")["global_bin"]:
        h = oracle.OracleHist([(n, 0.0, 1.0) for n in ex["nbins"]])
        assert h.global_bin(ex["b"]) == ex["g"], ex["cite"]


def test_spec_fill_bulk():
    ex = _load("spec_examples.json")["fill_bulk"][0]
    h = oracle.OracleHist([(ex["nbins"], ex["xmin"], ex["xmax"])]).fill([np.array(ex["x"])])
    r = h.read()
    for g, v in ex["content"].items():
        assert r["content"][int(g)] == v
    assert r["entries"] == ex["entries"]
    assert r["content"].sum() == len(ex["x"])


def test_spec_stats_update():
    for ex in _load("spec_examples.json")["stats_update"]:
        axes = ex.get("axes", [(10, 0.0, 1.0)] * ex["dim"])
        h = oracle.OracleHist([tuple(a) for a in axes]).fill([np.array(c) for c in ex["x"]], np.array(ex["w"]))
        np.testing.assert_array_equal(h.read()["stats"], np.array(ex["stats"]), err_msg=ex["cite"])


def test_spec_finalize_stats():
    for ex in _load("spec_examples.json")["finalize_stats"]:
        (m, s), = oracle.finalize_stats(ex["stats"], 1)
        assert m == ex["mean"] and s == ex["std"], ex["cite"]


def test_zero_weight_leaves_stats_unchanged():
    # (any x, w=0) -> acc unchanged; the bin still receives +0 and entries += 1
    h = oracle.OracleHist([(10, 0.0, 1.0)]).fill([np.array([0.33])], np.array([0.0]))
    r = h.read()
    assert np.all(r["stats"] == 0) and r["entries"] == 1 and r["content"].sum() == 0


# ------------------------------------------------------------------ IEEE pins (hand-derived)
def test_ieee_fixed_pins():
    for p in _load("ieee_pins.json")["pins"]:
        assert oracle.find_bin_fixed(p["nbins"], p["xmin"], p["xmax"], _x(p["x_hex"])) == p["bin"], p["why"]


def test_variable_pins():
    for p in _load("ieee_pins.json")["variable_pins"]:
        assert oracle.find_bin_variable(p["edges"], _x(p["x"])) == p["bin"], p["why"]


# ------------------------------------------------------------------ exact rational arithmetic
def _exact_bin(n, lo, hi, x):
    """1 + floor(n (x - lo) / (hi - lo)) in exact rational arithmetic on the double inputs."""
    q = Fraction(n) * (Fraction(x) - Fraction(lo)) / (Fraction(hi) - Fraction(lo))
    return q, 1 + math.floor(q)


def test_fixed_matches_exact_rational_away_from_integers():
    """PAPER.md:126's real formula: wherever the exact quotient is farther than 2^-40*max(q,1)
    from an integer, IEEE rounding (<= ~2 ulp) cannot move the floor, so the oracle's
    binary64 evaluation must equal the exact-rational floor."""
    rng = np.random.default_rng(1234)
    checked = 0
    for _ in range(3000):
        n = int(rng.choice([1, 2, 3, 7, 100, 1000, 12345, 10 ** 6, 2 ** 31 - 3]))
        lo = float(rng.uniform(-1e3, 1e3)) if rng.random() < 0.5 else 0.0
        width = float(10.0 ** rng.uniform(-6, 6))
        hi = lo + width
        if not lo < hi:
            continue
        for x in rng.uniform(lo, hi, size=8):
            x = float(x)
            if not (lo <= x < hi):
                continue
            q, b = _exact_bin(n, lo, hi, x)
            frac = q - math.floor(q)
            tol = Fraction(2) ** -40 * max(q, 1)
            if frac < tol or 1 - frac < tol:
                continue
            assert oracle.find_bin_fixed(n, lo, hi, x) == b, (n, lo, hi, x)
            checked += 1
    assert checked > 20000


def test_fixed_flow_routing():
    rng = np.random.default_rng(7)
    for _ in range(200):
        n = int(rng.integers(1, 5000))
        lo = float(rng.uniform(-10, 10))
        hi = lo + float(rng.uniform(1e-3, 10))
        for x in [lo - abs(rng.normal()) - 1e-9, np.nextafter(lo, -np.inf), hi, np.nextafter(hi, np.inf), hi + 5]:
            b = oracle.find_bin_fixed(n, lo, hi, float(x))
            assert b == (0 if x < lo else n + 1)
        b = oracle.find_bin_fixed(n, lo, hi, lo)
        assert b == 1


# ------------------------------------------------------------------ brute force (variable axes)
def _linear_scan(edges, x):
    """linear-scan oracle; flow per PAPER.md:126; bin = #edges <= x (reading R1)."""
    if x < edges[0]:
        return 0
    if not x < edges[-1]:
        return len(edges)
    return sum(1 for e in edges if e <= x)


def test_variable_matches_linear_scan_adversarial():
    rng = np.random.default_rng(99)
    for trial in range(300):
        n = int(rng.integers(1, 60))
        edges = np.cumsum(rng.uniform(1e-6, 1.0, size=n + 1)) - float(rng.uniform(0, 5))
        assert np.all(np.diff(edges) > 0)
        xs = list(rng.uniform(edges[0] - 1, edges[-1] + 1, size=20))
        for e in edges:   # every edge and +-1..3 ulps around it
            v = float(e)
            xs.append(v)
            up = dn = v
            for _ in range(3):
                up, dn = float(np.nextafter(up, np.inf)), float(np.nextafter(dn, -np.inf))
                xs += [up, dn]
        for x in xs:
            assert oracle.find_bin_variable(edges, float(x)) == _linear_scan(edges, float(x))


def test_fixed_equals_variable_on_uniform_edges_away_from_edges():
    """SPEC.md:124 property, restricted per DESIGN.md reading R3 to coordinates >= 4 ulps from
    every computed edge (it is false at the edges in floating point)."""
    rng = np.random.default_rng(5)
    for n, lo, hi in [(100, 0.0, 1.0), (1000, -1.0, 1.0), (37, 2.5, 9.75)]:
        edges = np.array([lo + i * (hi - lo) / n for i in range(n + 1)])
        edges[-1] = hi
        xs = rng.uniform(lo - 0.1, hi + 0.1, size=20000)
        h = oracle.OracleHist([(n, lo, hi)])
        hv = oracle.OracleHist([edges])
        gf = h.find_bins([xs])
        gv = hv.find_bins([xs])
        j = np.searchsorted(edges, xs)
        near = np.zeros(len(xs), bool)
        for k in (j - 1, j):
            kk = np.clip(k, 0, n)
            near |= np.abs(xs - edges[kk]) <= 4 * np.spacing(np.abs(edges[kk]) + np.abs(xs))
        assert np.array_equal(gf[~near], gv[~near])


# ------------------------------------------------------------------ global bin: bijection
def test_global_bin_bijection():
    for nb in ([3], [2, 3], [2, 1, 4]):
        h = oracle.OracleHist([(n, 0.0, 1.0) for n in nb])
        seen = set()
        for idx in np.ndindex(*[n + 2 for n in nb]):
            seen.add(h.global_bin(list(idx)))
        assert seen == set(range(int(np.prod([n + 2 for n in nb]))))


def test_global_bin_axis0_fastest():
    h = oracle.OracleHist([(2, 0.0, 1.0), (3, 0.0, 1.0), (4, 0.0, 1.0)])
    assert h.global_bin([1, 0, 0]) == 1
    assert h.global_bin([0, 1, 0]) == 4
    assert h.global_bin([0, 0, 1]) == 4 * 5


# ------------------------------------------------------------------ fill: conservation, stats
def test_conservation_and_stats_bruteforce_2d():
    rng = np.random.default_rng(11)
    n = 3000
    x = rng.uniform(-0.2, 1.2, n)
    y = rng.normal(0.5, 0.4, n)
    w = rng.uniform(-1, 2, n)
    h = oracle.OracleHist([(7, 0.0, 1.0), np.array([0.0, 0.1, 0.35, 0.5, 0.9, 1.0])]).fill([x, y], w)
    r = h.read()
    assert r["entries"] == n
    assert math.isclose(r["content"].sum(), math.fsum(w), rel_tol=0, abs_tol=1e-12 * np.abs(w).sum())
    assert math.isclose(r["sumw2"].sum(), math.fsum(w * w), rel_tol=1e-13)
    # brute force, exact rationals: in-range iff every axis bin in [1, n_a] (reading R6)
    e1 = [0.0, 0.1, 0.35, 0.5, 0.9, 1.0]
    inr = [(_exact_bin(7, 0.0, 1.0, float(a))[1] if 0 <= a < 1 else -1) in range(1, 8)
           and 1 <= _linear_scan(e1, float(b)) <= 5 for a, b in zip(x, y)]
    F = Fraction
    terms = {0: [], 1: [], 2: [], 3: [], 4: [], 5: [], 6: []}
    for a, b, ww, ok in zip(x, y, w, inr):
        if not ok:
            continue
        a, b, ww = F(float(a)), F(float(b)), F(float(ww))
        terms[0].append(ww); terms[1].append(ww * ww)
        terms[2].append(ww * a); terms[3].append(ww * a * a)
        terms[4].append(ww * b); terms[5].append(ww * b * b); terms[6].append(ww * a * b)
    for k in range(7):
        exact = float(sum(terms[k], F(0)))
        scale = float(sum((abs(t) for t in terms[k]), F(0)))
        # one or two roundings per term: |oracle - exact| <= ~2^-52 * sum|term|
        assert abs(r["stats"][k] - exact) <= 2.0 ** -50 * scale, k
        assert math.isclose(r["stats_abs"][k], scale, rel_tol=1e-12)


def test_unit_weight_counts_exact_and_stats_consistent():
    wl = bhgen.workload("C1", 200_000)
    x = wl.column(0, 0, wl.n_events)
    h = oracle.OracleHist([(100, 0.0, 1.0)]).fill([x])
    r = h.read()
    assert r["content"].sum() == wl.n_events == r["entries"]
    assert np.array_equal(r["content"], r["sumw2"])
    assert np.all(r["content"] == np.round(r["content"]))
    assert r["stats"][0] == r["content"][1:101].sum() == r["stats"][1]
    # independent count via exact rationals on a subsample of bins: numpy histogram on
    # points far from edges gives the same per-bin counts as the formula
    cnt, _ = np.histogram(x, bins=100, range=(0.0, 1.0))
    diff = np.abs(cnt - r["content"][1:101])
    assert diff.sum() <= 2 * np.sum(np.abs(x * 100 - np.round(x * 100)) < 1e-12)


def test_bulk_split_and_merge_invariance():
    # splitting into B fills (or merging partial states) changes nothing
    wl = bhgen.workload("C3", 60_000)
    x, y = wl.column(0, 0, wl.n_events), wl.column(1, 0, wl.n_events)
    ref = oracle.OracleHist([(50, 0.0, 1.0), (40, 0.0, 1.0)]).fill([x, y]).read()
    for B in (2, 7, 32):
        h = oracle.OracleHist([(50, 0.0, 1.0), (40, 0.0, 1.0)])
        cuts = np.linspace(0, wl.n_events, B + 1).astype(int)
        for a, b in zip(cuts[:-1], cuts[1:]):
            h.fill([x[a:b], y[a:b]])
        r = h.read()
        assert np.array_equal(r["content"], ref["content"]) and r["entries"] == ref["entries"]
        assert np.array_equal(r["stats"][[0, 1]], ref["stats"][[0, 1]])
        np.testing.assert_allclose(r["stats"], ref["stats"], rtol=1e-14)
    parts = []
    for r0 in range(4):
        a, b = bhgen.shard(wl.n_events, r0, 4)
        parts.append(oracle.OracleHist([(50, 0.0, 1.0), (40, 0.0, 1.0)]).fill([x[a:b], y[a:b]]))
    m = parts[0]
    for p in parts[1:]:
        m.merge(p)
    r = m.read()
    assert np.array_equal(r["content"], ref["content"]) and r["entries"] == ref["entries"]


def test_empty_fill():
    h = oracle.OracleHist([(10, 0.0, 1.0)]).fill([np.array([])])
    r = h.read()
    assert r["entries"] == 0 and r["content"].sum() == 0 and np.all(r["stats"] == 0)


def test_invalid_axes_rejected():
    with pytest.raises(ValueError):
        oracle.OracleHist([(0, 0.0, 1.0)])
    with pytest.raises(ValueError):
        oracle.OracleHist([(10, 1.0, 1.0)])
    with pytest.raises(ValueError):
        oracle.OracleHist([np.array([0.0, 0.5, 0.5, 1.0])])


# ------------------------------------------------------------------ closed-form moments
def _truncated_moments(pdf, lo, hi):
    from scipy import integrate
    p = integrate.quad(pdf, lo, hi, limit=500, points=[0.505, 0.5])[0]
    m = integrate.quad(lambda t: t * pdf(t), lo, hi, limit=500, points=[0.505, 0.5])[0] / p
    m2 = integrate.quad(lambda t: t * t * pdf(t), lo, hi, limit=500, points=[0.505, 0.5])[0] / p
    return p, m, math.sqrt(m2 - m * m)


def test_uniform_law_moments():
    # SPEC.md:461 acceptance 7 (mean 0.5, sigma 1/sqrt(12) within 1e-3), at 4e6 events
    wl = bhgen.workload("C1", 4_000_000)
    x = wl.column(0, 0, wl.n_events)
    r = oracle.OracleHist([(1000, 0.0, 1.0)]).fill([x]).read()
    (m, s), = oracle.finalize_stats(r["stats"], 1)
    assert r["content"].sum() == wl.n_events
    assert abs(m - 0.5) < 1e-3 and abs(s - 1 / math.sqrt(12)) < 1e-3


def test_gaussian_c2_moments_and_flow_fraction():
    from scipy import stats as sst
    wl = bhgen.workload("C2", 2_000_000)
    x = wl.column(0, 0, wl.n_events)
    w = wl.column(1, 0, wl.n_events)
    edges = wl.hists[0].axes[0].edges
    r = oracle.OracleHist([edges]).fill([x], w).read()
    p, mu, sd = _truncated_moments(lambda t: sst.norm.pdf(t, 0.5, 0.15), 0.0, 1.0)
    (m, s), = oracle.finalize_stats(r["stats"], 1)
    n = wl.n_events
    assert abs(m - mu) < 5 * sd / math.sqrt(n)
    assert abs(s - sd) < 5 * sd / math.sqrt(2 * n) + 1e-4
    # weights are independent of x: flow fraction from contents matches 1-P(in range)
    flow = (r["content"][0] + r["content"][-1]) / r["content"].sum()
    assert abs(flow - (1 - p)) < 5 * math.sqrt((1 - p) / n) + 5e-5
    assert abs(r["stats"][0] / r["stats"][1] - 1.0 / (13.0 / 12.0)) < 0.01  # E[w]/E[w^2] for U[.5,1.5)


def test_cauchy_c4_shape():
    from scipy import stats as sst
    wl = bhgen.workload("C4", 400_000)
    cols = [wl.column(a, 0, wl.n_events) for a in range(3)]
    r = oracle.OracleHist([(100, 0.0, 1.0)] * 3).fill(cols).read()
    p, mu, sd = _truncated_moments(lambda t: sst.cauchy.pdf(t, 0.505, 0.002), 0.0, 1.0)
    n_in = r["stats"][0]
    assert abs(n_in / wl.n_events - p ** 3) < 5 * math.sqrt(p ** 3 * (1 - p ** 3) / wl.n_events)
    m = r["stats"][2] / n_in
    assert abs(m - mu) < 5 * sd / math.sqrt(n_in)
    # hottest bin: P(central bin [0.5,0.51) per axis)^3
    pc = sst.cauchy.cdf(0.51, 0.505, 0.002) - sst.cauchy.cdf(0.5, 0.505, 0.002)
    hot = r["content"].max() / wl.n_events
    assert abs(hot - pc ** 3) < 5 * math.sqrt(pc ** 3 / wl.n_events)


# ------------------------------------------------------------------ Filter + Define oracle
def test_expr_oracle_hand_values():
    from oracle import expr
    x = np.array([3.0, -1.0, 0.5, np.nan])
    y = np.array([4.0, 2.0, 0.5, 1.0])
    prog = [("mul", 2, 0, 0, 0, 0.0), ("mul", 3, 1, 1, 0, 0.0), ("add", 4, 2, 3, 0, 0.0), ("sqrt", 5, 4, 0, 0, 0.0),
            ("const", 6, 0, 0, 0, 0.0), ("gt", 7, 0, 6, 0, 0.0)]
    r = expr.run_program([x, y], prog, 4)
    assert r[5][0] == 5.0 and r[5][1] == np.sqrt(5.0) and r[5][2] == np.sqrt(0.5)
    assert list(r[7][:3]) == [1.0, 0.0, 1.0] and r[7][3] == 0.0          # NaN > 0 is false
    h = expr.fill_expr([(10, 0.0, 10.0)], [x, y], prog, [5], filter_reg=7)
    out = h.read()
    assert out["entries"] == 2 and out["content"][6] == 1.0 and out["content"][1] == 1.0   # r=5 -> bin 6


# ------------------------------------------------------------------ association of the fixed formula
def _rn(q: Fraction) -> Fraction:
    """Round a rational to the nearest binary64 (ties to even) with integer arithmetic only —
    an emulation independent of the host FPU, for normal-range values."""
    if q == 0:
        return Fraction(0)
    s = -1 if q < 0 else 1
    q = abs(q)
    e = q.numerator.bit_length() - q.denominator.bit_length()
    while Fraction(2) ** e > q:
        e -= 1
    while Fraction(2) ** (e + 1) <= q:
        e += 1
    assert -1022 <= e <= 1023
    scaled = q / Fraction(2) ** (e - 52)           # in [2^52, 2^53)
    m, r = divmod(scaled.numerator, scaled.denominator)
    twice = 2 * r
    if twice > scaled.denominator or (twice == scaled.denominator and m % 2 == 1):
        m += 1
    return s * Fraction(m) * Fraction(2) ** (e - 52)


def _softfloat_bin(n, lo, hi, x):
    """Reading R2 evaluated with the rounding emulation: 1 + trunc(RN(RN(n*RN(x-lo)) / RN(hi-lo)))."""
    d = _rn(Fraction(x) - Fraction(lo))
    q = _rn(_rn(Fraction(n) * d) / _rn(Fraction(hi) - Fraction(lo)))
    return 1 + math.floor(q)


def test_association_pins():
    """Hand-derived pins on non-unit ranges where (n*d)/D, d*(n/D) and n*(d/D) give different
    bins (tests/golden/ieee_pins.json 'association_pins', PAPER.md:126 + reading R2). Each
    derivation is re-checked with the integer rounding emulation, then the oracle is held to it."""
    for p in _load("ieee_pins.json")["association_pins"]:
        x = _x(p["x_hex"])
        assert _softfloat_bin(p["nbins"], p["xmin"], p["xmax"], x) == p["bin"], p["why"]
        assert _exact_bin(p["nbins"], p["xmin"], p["xmax"], x)[1] == p["real_bin"], p["why"]
        assert oracle.find_bin_fixed(p["nbins"], p["xmin"], p["xmax"], x) == p["bin"], p["why"]


def test_fixed_softfloat_near_edges():
    """Every coordinate within 3 ulps of a computed edge on a few non-unit axes: the oracle equals
    the integer rounding emulation of reading R2 (where the associations disagree most)."""
    for n, lo, hi in [(100, 0.0, 3.0), (1000, -1.0, 2.0), (37, 0.1, 0.8), (7, -2.5, 9.75)]:
        D = hi - lo
        checked = 0
        for k in range(0, n + 1):
            x0 = lo + k * D / n
            xs = [x0]
            up = dn = x0
            for _ in range(3):
                up, dn = float(np.nextafter(up, np.inf)), float(np.nextafter(dn, -np.inf))
                xs += [up, dn]
            for x in xs:
                if not (lo < x < hi) or x - lo < 1e-300:
                    continue
                assert oracle.find_bin_fixed(n, lo, hi, x) == _softfloat_bin(n, lo, hi, x), (n, lo, hi, x)
                checked += 1
        assert checked > 5 * (n - 1)


def test_fixed_numpy_vectorized_1e7():
    """SURVEY §8(c) pin: an independent vectorised numpy evaluation of reading R2
    (numpy float64 ops are single IEEE roundings, never contracted) over 1.2e7 random and
    near-edge coordinates on 24 axes must agree with the oracle event by event."""
    rng = np.random.default_rng(2024)
    total = 0
    for t in range(24):
        n = int(rng.choice([3, 7, 100, 1000, 9973, 65536, 10 ** 6]))
        lo = float(rng.choice([0.0, -1.0, float(rng.uniform(-100, 100))]))
        hi = lo + float(rng.choice([1.0, 3.0, 0.3, float(10.0 ** rng.uniform(-3, 3))]))
        m = 250_000
        xs = rng.uniform(lo - 0.01 * (hi - lo), hi + 0.01 * (hi - lo), m)
        k = rng.integers(0, n + 1, m)
        e = lo + k * ((hi - lo) / n)
        sh = rng.integers(-3, 4, m)
        near = e.copy()
        for s in (1, 2, 3):
            near = np.where(sh >= s, np.nextafter(near, np.inf), near)
            near = np.where(sh <= -s, np.nextafter(near, -np.inf), near)
        x = np.concatenate([xs, near, [lo, hi, np.nan, -np.inf, np.inf, -0.0]])
        with np.errstate(invalid="ignore"):
            q = (np.float64(n) * (x - lo)) / (hi - lo)
            ref = np.where(x < lo, 0, np.where(~(x < hi), n + 1, 1 + np.trunc(np.where(x < lo, 0, q))))
        got = oracle.OracleHist([(n, lo, hi)]).find_bins([x])
        assert np.array_equal(got, ref.astype(np.int32)), (n, lo, hi)
        total += len(x)
    assert total >= 12_000_000


# ------------------------------------------------------------------ 3-D stats, exact rationals
def test_conservation_and_stats_bruteforce_3d():
    """All 11 GetStats sums of a TH3 (reading R8, PAPER.md:126 'depends on the dimension'):
    [Σw, Σw², Σwx, Σwx², Σwy, Σwy², Σwxy, Σwz, Σwz², Σwxz, Σwyz], each against an exact
    rational sum over the events that are in range on every axis. x, y, z have different
    laws so every cross term has a different value (swapping any two indices fails)."""
    rng = np.random.default_rng(33)
    n = 2500
    x = rng.uniform(-0.1, 1.1, n)
    y = rng.normal(2.0, 0.6, n)
    z = rng.exponential(3.0, n) - 1.0
    w = rng.uniform(-0.5, 2.0, n)
    ez = [-1.0, 0.0, 0.5, 2.0, 4.5, 8.0]
    h = oracle.OracleHist([(9, 0.0, 1.0), (6, 0.5, 3.5), np.array(ez)]).fill([x, y, z], w)
    r = h.read()
    assert r["entries"] == n and len(r["stats"]) == 11
    assert math.isclose(r["content"].sum(), math.fsum(w), rel_tol=0, abs_tol=1e-12 * np.abs(w).sum())
    F = Fraction
    terms = [[] for _ in range(11)]
    for a, b, c, ww in zip(x, y, z, w):
        a, b, c, ww = float(a), float(b), float(c), float(ww)
        if not (1 <= _exact_bin(9, 0.0, 1.0, a)[1] <= 9 if 0.0 <= a < 1.0 else False):
            continue
        if not (1 <= _exact_bin(6, 0.5, 3.5, b)[1] <= 6 if 0.5 <= b < 3.5 else False):
            continue
        if not 1 <= _linear_scan(ez, c) <= 5:
            continue
        A, B, C, W = F(a), F(b), F(c), F(ww)
        for k, t in enumerate([W, W * W, W * A, W * A * A, W * B, W * B * B, W * A * B,
                               W * C, W * C * C, W * A * C, W * B * C]):
            terms[k].append(t)
    assert 300 < len(terms[0]) < n
    for k in range(11):
        exact = float(sum(terms[k], F(0)))
        scale = float(sum((abs(t) for t in terms[k]), F(0)))
        assert abs(r["stats"][k] - exact) <= 2.0 ** -50 * scale, k
    # the cross terms are pairwise far apart, so an index swap cannot pass
    s = r["stats"]
    for i, j in [(6, 9), (6, 10), (9, 10), (7, 4), (8, 5), (2, 4), (2, 7)]:
        assert abs(s[i] - s[j]) > 1e-3 * max(abs(s[i]), abs(s[j])), (i, j)


def test_stats_hand_values_3d():
    """One in-range TH3 event (x, y, z) = (0.5, 2, 4), w = 3: the 11 sums by hand."""
    h = oracle.OracleHist([(10, 0.0, 1.0), (10, 0.0, 8.0), (10, 0.0, 8.0)])
    h.fill([np.array([0.5]), np.array([2.0]), np.array([4.0])], np.array([3.0]))
    # Σw=3, Σw²=9, Σwx=1.5, Σwx²=0.75, Σwy=6, Σwy²=12, Σwxy=3, Σwz=12, Σwz²=48, Σwxz=6, Σwyz=24
    assert list(h.read()["stats"]) == [3.0, 9.0, 1.5, 0.75, 6.0, 12.0, 3.0, 12.0, 48.0, 6.0, 24.0]


# ------------------------------------------------------------------ Filter + Define: every opcode
_NAN, _INF = float("nan"), float("inf")
# columns: a, b, c (registers 0, 1, 2)
_EA = [3.0, -2.0, _NAN, 0.0, -0.0, _INF]
_EB = [4.0, 0.5, 1.0, _NAN, 0.0, _INF]
_EC = [10.0, 20.0, 30.0, 40.0, 50.0, 60.0]
# Hand values per opcode (include/bhist.h BH_OP_*; IEEE 754 binary64 semantics: NaN compares
# false, fmin/fmax are minNum/maxNum so a NaN operand yields the other one, a truth value is
# "!= 0" so NaN is true, sqrt(-0) = -0).  '-0' marks a value whose sign bit must be set.
_EXPR_HAND = {
    "const": (("const", 3, 0, 0, 0, 2.5), [2.5] * 6),
    "copy": (("copy", 3, 0, 0, 0, 0.0), [3.0, -2.0, _NAN, 0.0, "-0", _INF]),
    "add": (("add", 3, 0, 1, 0, 0.0), [7.0, -1.5, _NAN, _NAN, 0.0, _INF]),
    "sub": (("sub", 3, 0, 1, 0, 0.0), [-1.0, -2.5, _NAN, _NAN, "-0", _NAN]),
    "mul": (("mul", 3, 0, 1, 0, 0.0), [12.0, -1.0, _NAN, _NAN, "-0", _INF]),
    "div": (("div", 3, 0, 1, 0, 0.0), [0.75, -4.0, _NAN, _NAN, _NAN, _NAN]),
    "sqrt": (("sqrt", 3, 0, 0, 0, 0.0), [1.7320508075688772, _NAN, _NAN, 0.0, "-0", _INF]),
    "abs": (("abs", 3, 0, 0, 0, 0.0), [3.0, 2.0, _NAN, 0.0, 0.0, _INF]),
    "neg": (("neg", 3, 0, 0, 0, 0.0), [-3.0, 2.0, _NAN, "-0", 0.0, -_INF]),
    "min": (("min", 3, 0, 1, 0, 0.0), [3.0, -2.0, 1.0, 0.0, None, _INF]),
    "max": (("max", 3, 0, 1, 0, 0.0), [4.0, 0.5, 1.0, 0.0, None, _INF]),
    "lt": (("lt", 3, 0, 1, 0, 0.0), [1.0, 1.0, 0.0, 0.0, 0.0, 0.0]),
    "le": (("le", 3, 0, 1, 0, 0.0), [1.0, 1.0, 0.0, 0.0, 1.0, 1.0]),
    "gt": (("gt", 3, 0, 1, 0, 0.0), [0.0, 0.0, 0.0, 0.0, 0.0, 0.0]),
    "ge": (("ge", 3, 0, 1, 0, 0.0), [0.0, 0.0, 0.0, 0.0, 1.0, 1.0]),
    "eq": (("eq", 3, 0, 1, 0, 0.0), [0.0, 0.0, 0.0, 0.0, 1.0, 1.0]),
    "ne": (("ne", 3, 0, 1, 0, 0.0), [1.0, 1.0, 1.0, 1.0, 0.0, 0.0]),
    "and": (("and", 3, 0, 1, 0, 0.0), [1.0, 1.0, 1.0, 0.0, 0.0, 1.0]),
    "or": (("or", 3, 0, 1, 0, 0.0), [1.0, 1.0, 1.0, 1.0, 0.0, 1.0]),
    "not": (("not", 3, 0, 0, 0, 0.0), [0.0, 0.0, 0.0, 1.0, 1.0, 0.0]),
    "select": (("select", 3, 0, 1, 2, 0.0), [4.0, 0.5, 1.0, 40.0, 50.0, _INF]),
}


def _check_hand(got, want, name):
    for i, (g, v) in enumerate(zip(got, want)):
        if v is None:                      # fmin(-0, +0): either zero is a valid minNum
            assert g == 0.0, (name, i)
        elif v == "-0":
            assert g == 0.0 and math.copysign(1.0, g) < 0, (name, i, g)
        elif isinstance(v, float) and math.isnan(v):
            assert math.isnan(g), (name, i, g)
        else:
            assert g == v and (v != 0.0 or math.copysign(1.0, g) > 0), (name, i, g, v)


def test_expr_every_opcode_hand_values():
    from oracle import expr
    from paper_2401_13310_b200.bhist import OPS   # names only (the opcode table of the header)
    assert set(_EXPR_HAND) == set(OPS)
    cols = [np.array(_EA), np.array(_EB), np.array(_EC)]
    for name, (op, want) in _EXPR_HAND.items():
        r = expr.run_program(cols, [op], 6)
        _check_hand(list(r[3]), want, name)
    # programs chain through registers in order, and the filter keeps exactly the truthy events:
    # r3 = b - a, r4 = r3*r3, r5 = (a == a) (false only for NaN); weights c
    prog = [("sub", 3, 1, 0, 0, 0.0), ("mul", 4, 3, 3, 0, 0.0), ("eq", 5, 0, 0, 0, 0.0)]
    h = expr.fill_expr([(4, 0.0, 100.0)], cols, prog, [4], weight_reg=2, filter_reg=5).read()
    # kept events 0,1,3,4,5: r4 = 1, 6.25, NaN (0-NaN), 0, NaN (inf-inf) -> bin 1 gets 10+20+50,
    # overflow (bin 5, NaN routed per reading R5) gets 40+60
    assert h["entries"] == 5
    assert h["content"][1] == 80.0 and h["content"][5] == 100.0 and h["content"].sum() == 180.0
