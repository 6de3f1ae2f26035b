#!/bin/bash
for lib in paper_2401_13310_b200/libbhist.so build_ab/libbhist_a1.so build_ab/libbhist_a2.so; do
BHIST_LIBRARY=$PWD/$lib timeout 300 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$lib C5 %.4g ev/s frac %.3f launch %.3f'%(d['value'], d['roofline']['frac'], d['roofline']['launch_ms']))"
BHIST_LIBRARY=$PWD/$lib python tools/peak_timing.py 2>&1 | grep " w " | awk '{print $1,$2,$5}' | tr '\n' ' '; echo
done
