timeout 900 python -m pytest tests/ -x -q -m "gpu" 2>&1 | tail -3
run() { python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 "$@" 2>>gpurun_out/b8.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config']['workload'][:36], d['config']['fill_strategy'][:20], '%.3g ev/s'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'launch_ms %.3f'%d['roofline']['launch_ms'], 'e2e %.3g'%d['e2e']['value'], 'launches', d['gpu_launches'], d['clocks']['sm_mhz'])
"; }
run --config C5
run --config C2
tail -2 gpurun_out/b8.err
