#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu --timeout=600 -x -k "peaked or fill_parity or tiny or fuzz or unaligned or f32 or expr or exact" > gpurun_out/pytest_cw.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_cw.log
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" "$@" 2>>gpurun_out/cw.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config']['workload'][:12], d['config']['fill_strategy'][:12], '%.4g ev/s'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'launch_ms %.3f'%d['roofline']['launch_ms'], 'ms/step %.3f'%d['ms_per_step'])
"; }
for c in C4W C3W C4; do run --config $c; done
run --config C3 --strategy cache
