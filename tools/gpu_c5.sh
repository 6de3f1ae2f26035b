timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m "gpu" -k "multi or C5" 2>&1 | tail -3
python bench.py --config C5 --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>&1 | tail -1 | cut -c 1-900
