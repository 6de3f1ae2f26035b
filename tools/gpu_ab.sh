#!/bin/bash
run() { timeout 300 env "$@" python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$C $*', '%.4g ev/s frac %.3f launch %.3f'%(d['value'], d['roofline']['frac'], d['roofline']['launch_ms']))"; }
C=C4W; run X=1; run BHIST_CACHE_SLOTS_W=8192; run BHIST_CACHE_SLOTS_W=2048
C=C3W; run X=1; run BHIST_CACHE_SLOTS_W=8192
C=C4; run X=1; run BHIST_CACHE_SLOTS_U=8192; run BHIST_CACHE_SLOTS_U=4096
C=C3; run X=1; run BHIST_SORT_CHUNK=268435456
C=C5; run X=1; run BHIST_CACHE_SLOTS_U=8192
