#!/bin/bash
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" "$@" 2>>gpurun_out/c5.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config']['workload'][:12], d['config']['fill_strategy'][:12], '%.4g ev/s'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'launch_ms %.3f'%d['roofline']['launch_ms'], 'ms/step %.3f'%d['ms_per_step'])
"; }
mkdir -p gpurun_out
run --config C5; run --config C5 --hist-strategy 6=sort; run --config C5 --hist-strategy 6=global
