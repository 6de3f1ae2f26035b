"""One small weighted fill (32768 events, 10k variable bins) repeated: ncu target."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2401_13310_b200 as pkg
rng = np.random.default_rng(3)
edges = np.concatenate([[0.0], np.cumsum(rng.uniform(0.5, 1.5, 10000))])
edges /= edges[-1]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
x = torch.rand(n, dtype=torch.float64, device="cuda")
w = torch.rand(n, dtype=torch.float64, device="cuda") + 0.5
mode = sys.argv[2] if len(sys.argv) > 2 else "var"
if mode == "var":
    h, cols = pkg.Histogram([edges]), [x]
else:
    h, cols = pkg.Histogram([(100, 0.0, 1.0)] * 2), [x, torch.rand(n, dtype=torch.float64, device="cuda")]
for _ in range(8):
    h.fill(cols, w)
torch.cuda.synchronize()
h.close()
