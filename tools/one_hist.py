"""Probe (not product code): fill one histogram of a workload a few times (for ncu):
python tools/one_hist.py C5 3 [log2 events]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bhgen
import oracle
import paper_2401_13310_b200 as pkg

name, hi = sys.argv[1], int(sys.argv[2])
n = 1 << int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 27
wl = bhgen.workload(name, n)
hist = wl.hists[hi]
cols = [torch.from_numpy(wl.column(c, 0, n)).cuda() for c in hist.cols]
w = torch.from_numpy(wl.column(wl.wcol, 0, n)).cuda() if hist.weighted else None
h = pkg.Histogram(oracle.oracle_axes(hist))
for _ in range(4):
    h.fill(cols, w)
torch.cuda.synchronize()
print("strategy", h.strategy(hist.weighted), "entries", h.read()["entries"])
