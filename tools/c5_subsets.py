"""Timing probe (not product code): subsets of C5's histograms that share columns, filled by
the one-pass kernel (BH_MULTI_ONE_PASS) vs one bh_fill pass per histogram."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bhgen
import oracle
import paper_2401_13310_b200 as pkg

n = 1 << 27
wl = bhgen.workload("C5", n)
cols = [torch.from_numpy(wl.column(c, 0, n)).cuda() for c in range(len(wl.columns))]
w = torch.from_numpy(wl.column(wl.wcol, 0, n)).cuda()


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


for sub in ([1, 2], [4, 7], [0, 5], [0, 4], [1, 2, 3], [0, 4, 5, 7], [1, 2, 6], [3, 6], [0, 1, 2, 3, 4]):
    hs = [pkg.Histogram(oracle.oracle_axes(wl.hists[i])) for i in sub]
    spec = ([wl.hists[i].cols for i in sub], [wl.hists[i].weighted for i in sub])
    solo = 0.0
    for h, i in zip(hs, sub):
        hist = wl.hists[i]
        solo += timed(lambda: h.fill([cols[c] for c in hist.cols], w if hist.weighted else None))
    pkg.bh_set_debug(hs[0].h, pkg.BH_DEBUG_REQUIRE_JIT)
    try:
        one = timed(lambda: pkg.fill_multi(hs, spec[0], spec[1], cols, w, mode=pkg.BH_MULTI_ONE_PASS))
    except Exception as e:
        one = float("nan")
        print("  one-pass failed:", e)
    print(f"H{sub}: solo passes {solo:6.3f} ms   one pass {one:6.3f} ms", flush=True)
    for h in hs:
        h.close()
