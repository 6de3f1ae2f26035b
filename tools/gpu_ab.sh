#!/bin/bash
run() { timeout 300 env "$@" python bench.py --config C1 --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('C1 $*', '%.4g ev/s frac %.3f launch %.4f'%(d['value'], d['roofline']['frac'], d['roofline']['launch_ms']))"; }
for e in 4 8 16 32 64; do run BHIST_PRIV_EPT=$e; done
for e in 8 32; do BHIST_PRIV_EPT=$e python tools/small_fill.py 2>&1 | head -2 | sed "s/^/ept=$e /"; done
