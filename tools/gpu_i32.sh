#!/bin/bash
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_abi.py -q -m gpu -x -k "i32 or f32 or abi" 2>&1 | tail -2
