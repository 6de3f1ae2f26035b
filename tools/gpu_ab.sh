#!/bin/bash
timeout 300 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "C1F,C2F" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print({k:(round(v['events_per_s']/1e9,1), round(v['frac'],3), round(v['fill_ms'],3)) for k,v in d['secondary'].items()})"
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py -q -m gpu -x -k "f32 or i32 or expr or fuzz" 2>&1 | tail -1
