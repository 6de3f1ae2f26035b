#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu --timeout=600 > gpurun_out/pytest_div.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_div.log; grep -E "^FAILED|^E  " gpurun_out/pytest_div.log | head -10
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" "$@" 2>>gpurun_out/d.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config']['workload'][:12], d['config']['fill_strategy'][:12], '%.4g ev/s'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'launch_ms %.3f'%d['roofline']['launch_ms'], 'ms/step %.3f'%d['ms_per_step'])
"; }
for c in C1S C2 C3 C4 C5; do run --config $c; done
run --config C3 --strategy cache
