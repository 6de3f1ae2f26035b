timeout 900 python -m pytest tests/ -x -q -m "gpu" 2>&1 | tail -1
for i in 1 2; do python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('C2 %.4g ev/s frac %.3f'%(d['value'], d['roofline']['frac']))"; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5c.csv python bench.py --config C5 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
python bench.py --config C4W --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline --strategy global 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('C4W global %.4g ev/s frac %.3f'%(d['value'], d['roofline']['frac']))"
python bench.py --config C4W --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('C4W auto %.4g ev/s frac %.3f'%(d['value'], d['roofline']['frac']))"
