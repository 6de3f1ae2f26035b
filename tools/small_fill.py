"""Latency probe for small fills (the paper's bulk size is 32768 events):
average time per bh_fill call over back-to-back calls on one stream (includes the
Python/ctypes call overhead), for 1D fixed unit, 1D variable weighted and 2D weighted."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2401_13310_b200 as pkg

rng = np.random.default_rng(3)
edges = np.concatenate([[0.0], np.cumsum(rng.uniform(0.5, 1.5, 10000))])
edges /= edges[-1]
for label, axes, ncol, weighted in (("TH1D 100 unit", [(100, 0.0, 1.0)], 1, False),
                                    ("TH1D 10k var w", [edges], 1, True),
                                    ("TH2D 100x100 w", [(100, 0.0, 1.0)] * 2, 2, True)):
    for n in (32768, 1 << 20):
        cols = [torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(ncol)]
        w = torch.rand(n, dtype=torch.float64, device="cuda") + 0.5 if weighted else None
        h = pkg.Histogram(axes)
        for _ in range(10):
            h.fill(cols, w)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 200
        e0.record()
        for _ in range(reps):
            h.fill(cols, w)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / reps
        print(f"{label:16s} n={n:8d}  {us:7.2f} us/fill  {n / us * 1e-3:8.3f} G ev/s", flush=True)
        h.close()
