"""Timing probe (not product code): each C5 histogram filled alone from the device-resident
C5 columns, under several environment settings (the planner reads BHIST_* at every call),
plus the whole set through bh_fill_multi.  Usage: python tools/c5_hists.py [log2 events] [env sets]
env sets: ';'-separated, each ','-separated K=V (empty = defaults)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bhgen
import oracle
import paper_2401_13310_b200 as pkg

n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
sets = (sys.argv[2] if len(sys.argv) > 2 else ";BHIST_NO_WARP_CACHE=1").split(";")
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


for st in sets:
    env = dict(kv.split("=", 1) for kv in st.split(",") if kv)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    tot = 0.0
    print(f"== [{st}]  n = {n}", flush=True)
    for i, hist in enumerate(wl.hists):
        h = pkg.Histogram(oracle.oracle_axes(hist))
        hc = [cols[c] for c in hist.cols]
        hw = w if hist.weighted else None
        ms = timed(lambda: h.fill(hc, hw))
        tot += ms
        bpe = 8 * (len(hist.cols) + hist.weighted)
        print(f"H{i} cols {hist.cols} w={int(hist.weighted)} G={h.nbins_total:8d} "
              f"strat {h.strategy(hist.weighted)}  {ms:7.3f} ms  {n / ms / 1e6:7.1f} Gev/s  frac {n * bpe / ms / 1e6 / 6550:5.3f}",
              flush=True)
        h.close()
    hs = [pkg.Histogram(oracle.oracle_axes(hist)) for hist in wl.hists]
    ms = timed(lambda: pkg.fill_multi(hs, [hh.cols for hh in wl.hists], [hh.weighted for hh in wl.hists], cols, w))
    for h in hs:
        h.close()
    print(f"sum of solo {tot:7.3f} ms   fill_multi {ms:7.3f} ms  (HBM floor {n * 56 / 6550e6:6.3f} ms)", flush=True)
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
