"""Debug probe (not product code): one bulk session on a tiny histogram, errors printed."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2401_13310_b200 as pkg

h = pkg.Histogram([(10, 0.0, 1.0)])
x = torch.full((1000,), 0.55, dtype=torch.float64).pin_memory()
print("pinned", x.is_pinned(), flush=True)
h.bulk_begin(False, timeout_ms=2000)
t0 = time.time()
try:
    h.bulk_fill([x])
    print("fill ok", time.time() - t0, flush=True)
    h.bulk_end()
    print("end ok", flush=True)
except Exception as e:
    print("ERR", e, flush=True)
try:
    torch.cuda.synchronize()
    print("sync ok", flush=True)
except Exception as e:
    print("SYNC ERR", e, flush=True)
print(h.read()["content"])

# the bench's P32K shape: 1000 random-width variable bins, bulks of 32768 pinned slices
import bhgen
edges = bhgen.edges_random_widths(bhgen.seed_of(6, 15), 1000)
total, bulk = 1 << 22, 32768
host = torch.empty(total, dtype=torch.float64).pin_memory()
bhgen.fill_ptr(bhgen.UNIFORM, bhgen.seed_of(6, 0), 0, total, 0.0, 1.0, host.data_ptr())
for axes in ([(1000, 0.0, 1.0)], [edges]):
    H = pkg.Histogram(axes)
    print("strategy", H.strategy(False), flush=True)
    H.bulk_begin(False, timeout_ms=3000)
    t0 = time.time()
    k = 0
    try:
        for i in range(0, total, bulk):
            H.bulk_fill([host[i:i + bulk]])
            k += 1
        H.bulk_end()
        print("ok", k, "bulks", (time.time() - t0) / k * 1e6, "us/bulk", H.read()["entries"], flush=True)
    except Exception as e:
        print("ERR after", k, "bulks:", e, flush=True)
        try:
            torch.cuda.synchronize(); print("sync ok")
        except Exception as e2:
            print("SYNC ERR", e2)
