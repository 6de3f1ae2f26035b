timeout 1200 python -m pytest tests/test_fuzz_gpu.py -q -m "gpu" --timeout=300 -x 2>&1 | tail -15
timeout 900 python -m pytest tests/test_parity_gpu.py -q -m "slow" --timeout=600 -k "2_31" 2>&1 | tail -3
