"""Small fills of every kernel family, for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bhgen  # noqa: E402
import paper_2401_13310_b200 as pkg  # noqa: E402

dev = "cuda:0"
rng = np.random.default_rng(1)
n = 20_011
for name in ("C1", "C2", "C3W", "C4"):
    wl = bhgen.workload(name, n)
    h = wl.hists[0]
    cols = [torch.from_numpy(wl.column(c, 0, n)).to(dev) for c in h.cols]
    w = torch.from_numpy(wl.column(wl.wcol, 0, n)).to(dev) if h.weighted else None
    for s in (pkg.BH_STRATEGY_PRIV, pkg.BH_STRATEGY_GLOBAL, pkg.BH_STRATEGY_CACHE):
        if s == pkg.BH_STRATEGY_PRIV and name in ("C3W", "C4"):
            continue
        H = pkg.Histogram(h.axes_spec(), strategy=s)
        H.fill(cols, w)
        H.fill([c[1:] for c in cols], None if w is None else w[1:])   # peeled / misaligned path
        H.find_bins(cols)
        H.read()
        H.close()
# SORT strategy: pass 1 (TMA-staged), plan, pass 2; several chunks and a partial last tile
os.environ["BHIST_SORT_CHUNK"] = "8192"
for name in ("C3", "C3W", "C4"):
    wl = bhgen.workload(name, n)
    h = wl.hists[0]
    cols = [torch.from_numpy(wl.column(c, 0, n)).to(dev) for c in h.cols]
    w = torch.from_numpy(wl.column(wl.wcol, 0, n)).to(dev) if h.weighted else None
    H = pkg.Histogram(h.axes_spec(), strategy=pkg.BH_STRATEGY_SORT)
    H.fill(cols, w)
    H.fill([c[1:] for c in cols], None if w is None else w[1:])   # unaligned: thread-loaded tiles
    H.read()
    H.close()
# peaked weighted 2D histograms: per-warp hot-bin caches (1 and several replicas)
y = torch.from_numpy(rng.normal(0.5, 0.05, n)).to(dev)
xp = torch.from_numpy(0.505 + 0.002 * np.tan(np.pi * (rng.random(n) - 0.5))).to(dev)
wp = torch.from_numpy(rng.uniform(0.5, 1.5, n)).to(dev)
for nb in (10, 100):
    H = pkg.Histogram([(nb, 0.0, 1.0), (nb, 0.0, 1.0)])
    H.fill([xp, y], wp)
    H.read()
    H.close()
# peaked weighted small histogram: replicas + collision-adaptive CAS
x = torch.from_numpy(0.505 + 0.002 * np.tan(np.pi * (rng.random(n) - 0.5))).to(dev)
w = torch.from_numpy(rng.uniform(0.5, 1.5, n)).to(dev)
H = pkg.Histogram([(100, 0.0, 1.0)])
H.fill([x], w)
H.read()
H.close()
# AUTO's device probes and the kernels they gate, on small inputs (BHIST_AUTO_MIN_EVENTS):
# GLOBAL paired REDs (C3W), CACHE + lane window (C4W), PRIVA + lane window (C5 H7), the unit
# WINDOW box (C5 H6, and a 1-D 200k-bin Gaussian), SORT (C3)
os.environ["BHIST_AUTO_MIN_EVENTS"] = "1"
na = 40_009
for name, hidx in (("C3W", 0), ("C4W", 0), ("C5", 7), ("C5", 6), ("C3", 0)):
    wl = bhgen.workload(name, na)
    h = wl.hists[hidx]
    cols = [torch.from_numpy(wl.column(c, 0, na)).to(dev) for c in h.cols]
    w = torch.from_numpy(wl.column(wl.wcol, 0, na)).to(dev) if h.weighted else None
    H = pkg.Histogram(h.axes_spec())
    H.fill(cols, w)
    H.fill(cols, w)
    H.read()
    H.close()
xg = torch.from_numpy(rng.normal(0.5, 0.15, na)).to(dev)
H = pkg.Histogram([(200_000, 0.0, 1.0)])
H.fill([xg])
H.read()
H.close()
del os.environ["BHIST_AUTO_MIN_EVENTS"]
# fused multi-histogram fill and the host path
wl = bhgen.workload("C5", n)
cols = [torch.from_numpy(wl.column(c, 0, n)).to(dev) for c in range(len(wl.columns))]
hs = [pkg.Histogram(h.axes_spec()) for h in wl.hists]
pkg.fill_multi(hs, [h.cols for h in wl.hists], [h.weighted for h in wl.hists], cols, cols[wl.wcol])
for H in hs:
    H.read()
    H.close()
# the one-pass fused kernel (NVRTC) of the same set
hs = [pkg.Histogram(h.axes_spec()) for h in wl.hists]
pkg.bh_set_debug(hs[0].h, pkg.BH_DEBUG_REQUIRE_JIT)
pkg.fill_multi(hs, [h.cols for h in wl.hists], [h.weighted for h in wl.hists], cols, cols[wl.wcol],
               mode=pkg.BH_MULTI_ONE_PASS)
for H in hs:
    H.read()
    H.close()
# the persistent bulk consumer: TMA-staged (C2 axis, weighted) and direct loads (large PRIV state),
# pinned and pageable bulks, bulks in flight
wl = bhgen.workload("C2", n)
xs, ws = wl.column(0, 0, n), wl.column(wl.wcol, 0, n)
for axes in (wl.hists[0].axes_spec(), [(13000, 0.0, 1.0)]):
    H = pkg.Histogram(axes)
    H.bulk_begin(True, timeout_ms=20000)
    t = 0
    for a in range(0, n, 3001):
        b = min(n, a + 3001)
        if a % 2:
            t = H.bulk_submit([torch.from_numpy(xs[a:b]).pin_memory()], torch.from_numpy(ws[a:b]).pin_memory())
        else:
            H.bulk_fill([np.ascontiguousarray(xs[a:b])], np.ascontiguousarray(ws[a:b]))
    H.bulk_wait(t)
    H.bulk_end()
    H.read()
    H.close()
H = pkg.Histogram([(1000, 0.0, 1.0)])
pkg.bh_set_chunk(H.h, 4096)
H.fill_host([torch.from_numpy(rng.random(n)).pin_memory()])
buf = H.pack()
H.unpack(buf)
H.read()
H.close()
torch.cuda.synchronize()
print("sanitize run ok")
