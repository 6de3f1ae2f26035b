"""Debug: SORT fill of a C3W-shaped workload at a given size, checked against CACHE."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bhgen
import oracle
import paper_2401_13310_b200 as pkg

n = int(sys.argv[1])
name = sys.argv[2] if len(sys.argv) > 2 else "C3W"
wl = bhgen.workload(name, n)
hist = wl.hists[0]
axes = oracle.oracle_axes(hist)
cols = [torch.from_numpy(wl.column(c, 0, n)).cuda() for c in hist.cols]
w = torch.from_numpy(wl.column(wl.wcol, 0, n)).cuda() if hist.weighted else None
res = {}
for s in (pkg.BH_STRATEGY_CACHE, pkg.BH_STRATEGY_SORT):
    h = pkg.Histogram(axes, strategy=s)
    h.fill(cols, w)
    res[s] = h.read()
    torch.cuda.synchronize()
    h.close()
a, b = res[pkg.BH_STRATEGY_CACHE], res[pkg.BH_STRATEGY_SORT]
print(n, name, "entries", a["entries"], b["entries"], "maxdiff", float(np.max(np.abs(a["content"] - b["content"]))))
