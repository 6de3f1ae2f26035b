python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m "gpu and not slow" 2>&1 | tail -3
run() { python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 "$@" 2>>gpurun_out/b2.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config']['workload'][:36], d['config']['fill_strategy'], '%.3g ev/s'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'launch_ms %.3f'%d['roofline']['launch_ms'], d['clocks']['sm_mhz'])
"; }
run --config C2
run --config C1S
run --config C3
run --config C3 --strategy cache
run --config C3W
run --config C4 --strategy cache
run --config C4W --strategy cache
tail -3 gpurun_out/b2.err
