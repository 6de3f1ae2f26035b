"""Filter + Define: fused in the fill (bh_fill_expr) vs materialized with torch then bh_fill."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_13310_b200 as pkg  # noqa: E402

n = 1 << 28
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
y = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
P = pkg.Program(2)
r = P.sqrt(P.add(P.mul(0, 0), P.mul(1, 1)))
cut = P.land(P.gt(0, P.const(-0.5)), P.lt(1, P.const(1.2)))
axes = [(100, 0.0, 3.0)]


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


h1 = pkg.Histogram(axes)
t_fused = timeit(lambda: (h1.reset(), pkg.fill_expr(h1, [x, y], P, [r], -1, cut)))
h2 = pkg.Histogram(axes)


def materialized():
    h2.reset()
    m = (x > -0.5) & (y < 1.2)
    rr = torch.sqrt(x[m] * x[m] + y[m] * y[m]).contiguous()
    h2.fill([rr])


t_mat = timeit(materialized)
a, b = h1.read(), h2.read()
assert a["entries"] == b["entries"] and np.array_equal(a["content"], b["content"])
print(f"events {n}: fused Filter+Define+fill {t_fused:.3f} ms ({n / t_fused / 1e6:.3g} G ev/s, "
      f"{16 * n / t_fused / 1e6:.0f} GB/s of input); torch-materialized {t_mat:.3f} ms -> {t_mat / t_fused:.1f}x")
