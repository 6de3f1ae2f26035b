#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu --timeout=300 -x -k "probe or strategy_resolution or sort or full_size" > gpurun_out/pytest_p.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_p.log
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" "$@" 2>>gpurun_out/p.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config']['workload'][:12], d['config']['fill_strategy'][:12], '%.4g ev/s'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'launch_ms %.3f'%d['roofline']['launch_ms'], 'ms/step %.3f'%d['ms_per_step'], 'e2e %.3g'%d['e2e']['value'])
"; }
for c in C3 C3W C4 C4W C5; do run --config $c; done
