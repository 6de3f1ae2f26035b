timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m "gpu and not slow" 2>&1 | tail -3
run() { python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 "$@" 2>>gpurun_out/b3.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config']['workload'][:36], d['config']['fill_strategy'], '%.3g ev/s'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'launch_ms %.3f'%d['roofline']['launch_ms'], d['clocks']['sm_mhz'])
"; }
for s in 0 2 3 4; do echo split8=$s; BHIST_L2_SPLIT8=$s run --config C2; done
run --config C1S
run --config C1
tail -3 gpurun_out/b3.err
