#!/bin/bash
for c in C3 C4 C2 C1S C5; do for lib in paper_2401_13310_b200/libbhist.so build_ab/libbhist_v.so; do
BHIST_LIBRARY=$PWD/$lib timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$lib $c %.4g ev/s frac %.3f launch %.3f'%(d['value'], d['roofline']['frac'], d['roofline']['launch_ms']))"; done; done
BHIST_LIBRARY=$PWD/build_ab/libbhist_v.so timeout 600 python -m pytest tests/test_parity_gpu.py -q -m gpu -x -k "find_bins or fill_parity" 2>&1 | tail -1
