#!/bin/bash
for c in C3W C3 C4W; do for st in cache global; do
timeout 300 python bench.py --config $c --strategy $st --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$st $c %.4g ev/s frac %.3f launch %.3f'%(d['value'], d['roofline']['frac'], d['roofline']['launch_ms']))"; done; done
