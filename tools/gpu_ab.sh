#!/bin/bash
run() { timeout 300 env "$@" python bench.py --config $C --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$C $*', '%.4g ev/s frac %.3f launch %.4f'%(d['value'], d['roofline']['frac'], d['roofline']['launch_ms']))"; }
C=C1; for r in 32 16 8 4 1; do run BHIST_PRIV_REPLICAS=$r; done
C=C1S; for r in 32 16 8; do run BHIST_PRIV_REPLICAS=$r; done
