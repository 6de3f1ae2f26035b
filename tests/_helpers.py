"""Shared test helpers: run the CUDA path (through the C ABI) and the oracle on the same
seeded bytes, and compare with the tolerances of BASELINE.json's north star:
bin indices bit-exact, unit-weight counts exact, weighted sums within 1e-12 relative
(relative to sum|term|, reading R14)."""
import multiprocessing as mp

import numpy as np

import bhgen
import oracle

RTOL = 1e-12


def gen_columns(wl, hist, start, n):
    cols = [wl.column(c, start, n) for c in hist.cols]
    w = wl.column(wl.wcol, start, n) if hist.weighted else None
    return cols, w


def compare(got, ref, weighted, what=""):
    assert got["entries"] == ref["entries"], (what, got["entries"], ref["entries"])
    if not weighted:
        assert np.array_equal(got["content"], ref["content"]), (what, np.flatnonzero(got["content"] != ref["content"])[:10])
        assert np.array_equal(got["sumw2"], ref["sumw2"]), what
        assert got["stats"][0] == ref["stats"][0] and got["stats"][1] == ref["stats"][1], what
    else:
        dc = np.abs(got["content"] - ref["content"])
        bad = dc > RTOL * ref["abs_content"]
        assert not bad.any(), (what, np.flatnonzero(bad)[:10], dc[bad][:5], ref["abs_content"][bad][:5])
        ds = np.abs(got["sumw2"] - ref["sumw2"])
        assert not (ds > RTOL * ref["sumw2"]).any(), what
    dst = np.abs(got["stats"] - ref["stats"])
    assert not (dst > RTOL * ref["stats_abs"]).any(), (what, got["stats"], ref["stats"], dst / np.maximum(ref["stats_abs"], 1e-300))


def _oracle_worker(args):
    name, n_total, hidx, start, n, chunk = args
    wl = bhgen.workload(name, n_total)
    hist = wl.hists[hidx]
    h = oracle.OracleHist(oracle.oracle_axes(hist))
    for off in range(start, start + n, chunk):
        m = min(chunk, start + n - off)
        cols, w = gen_columns(wl, hist, off, m)
        h.fill(cols, w)
    return h.read()


def oracle_parallel(name, n_total, hidx=0, start=0, n=None, nproc=None, chunk=1 << 22):
    """The oracle over [start, start+n) split into nproc contiguous shards, merged by
    summation (exact for counts; weighted sums gain <= nproc roundings ~1e-16)."""
    n = n_total if n is None else n
    nproc = nproc or max(1, min(16, mp.cpu_count()))
    bounds = [(start + (n * r) // nproc, start + (n * (r + 1)) // nproc) for r in range(nproc)]
    jobs = [(name, n_total, hidx, a, b - a, chunk) for a, b in bounds if b > a]
    ctx = mp.get_context("fork")
    with ctx.Pool(len(jobs)) as pool:
        parts = pool.map(_oracle_worker, jobs)
    out = {k: sum((p[k] for p in parts[1:]), parts[0][k].copy() if hasattr(parts[0][k], "copy") else parts[0][k])
           for k in parts[0]}
    return out
