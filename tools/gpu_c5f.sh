timeout 900 python -m pytest tests/ -q -m "gpu" --timeout=300 2>&1 | grep -E "passed|failed|error|FAIL" | tail -15
timeout 300 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('C5 %.4g ev/s ms %.3f'%(d['value'], d['ms_per_step']))"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('C2 %.4g ev/s frac %.3f'%(d['value'], d['roofline']['frac']))"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5f.csv python bench.py --config C5 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
