#!/bin/bash
# A/B of two library builds on the default C2 bench (alternating, 2 runs each)
for i in 1 2; do for lib in paper_2401_13310_b200/libbhist.so build_ab/libbhist_split.so; do
BHIST_LIBRARY=$PWD/$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$lib C2 %.4g ev/s frac %.3f'%(d['value'], d['roofline']['frac']))"; done; done
BHIST_LIBRARY=$PWD/build_ab/libbhist_split.so timeout 600 python -m pytest tests/test_parity_gpu.py -q -m gpu -x -k "C2 and fill_parity" 2>&1 | tail -1
