#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu --timeout=300 -x -k "guide or find_bins or multi or fill_parity or fuzz" > gpurun_out/pytest_g.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_g.log
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" "$@" 2>>gpurun_out/g.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config']['workload'][:12], d['config']['fill_strategy'][:12], '%.4g ev/s'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'launch_ms %.3f'%d['roofline']['launch_ms'], 'e2e %.3g'%d['e2e']['value'], 'pcie_frac %.3f'%d['e2e']['pcie_frac'])
"; }
run --config C5; run --config C2
