timeout 900 python -m pytest tests/ -q -m "gpu" --timeout=300 2>&1 | grep -E "passed|failed" | tail -3
timeout 600 python bench.py --steps 20 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('C2 %.4g ev/s frac %.3f e2e %.3g clocks %s' % (d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks']))
for k,v in d['secondary'].items(): print(k, '%.4g ev/s frac %.3f bpe %d %s' % (v['events_per_s'], v['frac'], v['bytes_per_event'], v['fill_strategy']))
"
