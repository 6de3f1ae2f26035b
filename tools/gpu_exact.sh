timeout 900 python -m pytest tests/ -q -m "gpu" --timeout=300 2>&1 | grep -E "passed|failed" | tail -2
for c in C2 C3W C4W; do timeout 300 python bench.py --config $c --strategy exact --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$c exact %.4g ev/s frac %.3f launch_ms %.3f'%(d['value'], d['roofline']['frac'], d['roofline']['launch_ms']))"; done
