"""Timing probe: weighted 2D fills of Cauchy-peaked x (C5's c4) and N(0.5,0.05) y (c5)
for several bin counts -> how the PRIV/PRIVA sink scales with replicas / contention."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2401_13310_b200 as pkg

n = 1 << 27
g = torch.Generator(device="cuda").manual_seed(1)
u = torch.rand(n, device="cuda", dtype=torch.float64, generator=g)
x = 0.505 + 0.002 * torch.tan(np.pi * (u - 0.5))
y = 0.5 + 0.05 * torch.randn(n, device="cuda", dtype=torch.float64, generator=g)
w = 0.5 + torch.rand(n, device="cuda", dtype=torch.float64, generator=g)
ux = torch.rand(n, device="cuda", dtype=torch.float64, generator=g)
uy = torch.rand(n, device="cuda", dtype=torch.float64, generator=g)
for label, cx, cy in (("peaked", x, y), ("uniform", ux, uy)):
    for nb in (10, 30, 50, 70, 100):
        for weighted in (True, False):
            h = pkg.Histogram([(nb, 0.0, 1.0), (nb, 0.0, 1.0)])
            ww = w if weighted else None
            for _ in range(3):
                h.fill([cx, cy], ww)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                h.fill([cx, cy], ww)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            print(f"{label:8s} {nb:4d}^2 {'w' if weighted else 'u'} {ms:7.3f} ms  {n / ms / 1e6:8.3g} Gev/s  strat {h.strategy(weighted)}", flush=True)
            h.close()
