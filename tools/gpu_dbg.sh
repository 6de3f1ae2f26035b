#!/bin/bash
for n in 70000000 200000000; do timeout 300 python tools/sort_debug.py $n C3W 2>&1 | grep -v "^frame" | tail -1; timeout 300 python tools/sort_debug.py $n C3 2>&1 | grep -v "^frame" | tail -1; done
timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu --timeout=300 -x -k "sort" 2>&1 | tail -2
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" "$@" 2>>gpurun_out/sort.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config']['workload'][:12], d['config']['fill_strategy'][:12], '%.4g ev/s'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'launch_ms %.3f'%d['roofline']['launch_ms'], 'ms/step %.3f'%d['ms_per_step'], 'e2e %.3g'%d['e2e']['value'])
"; }
for c in C3 C3W; do run --config $c --strategy sort; done
