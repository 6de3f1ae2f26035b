timeout 900 python -m pytest tests/ -q -m "gpu" --timeout=300 -x 2>&1 | grep -E "passed|failed|error|FAIL" | tail -8
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" "$@" 2>>gpurun_out/st.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config']['workload'][:26], d['config']['fill_strategy'][:8], '%.4g ev/s'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'launch_ms %.3f'%d['roofline']['launch_ms'])
"; }
for c in C3 C3W C4 C4W; do echo "-- $c"; run --config $c; BHIST_NO_STAGE=1 run --config $c; run --config $c --strategy global; done
tail -3 gpurun_out/st.err
