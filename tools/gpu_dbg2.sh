#!/bin/bash
for i in 1 2 3 4 5 6; do
timeout 300 python -m pytest tests/test_parity_gpu.py -q -m gpu -k "peaked" 2>&1 | tail -1
done
bash tools/gpu_cw.sh
