timeout 600 python -m pytest tests/ -x -q -m "gpu" -p pytest_timeout --timeout=120 2>&1 | tail -1
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 "$@" 2>>gpurun_out/b11.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config']['workload'][:30], d['config']['fill_strategy'][:12], '%.4g ev/s'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'launch_ms %.3f'%d['roofline']['launch_ms'])
"; }
run --config C2
BHIST_PRIV_REPLICAS=1 run --config C1S
run --config C1S
run --config C1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5d.csv python bench.py --config C5 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
tail -2 gpurun_out/b11.err
