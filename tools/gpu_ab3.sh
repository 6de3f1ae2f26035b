for lib in build_ab/libbhist_prev2.so build_ab/libbhist_vm.so paper_2401_13310_b200/libbhist.so; do
BHIST_LIBRARY=$PWD/$lib timeout 600 python bench.py --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$lib C2 %.4g ev/s frac %.3f' % (d['value'], d['roofline']['frac']))
for k,v in d['secondary'].items(): print('   ', k, '%.4g ev/s frac %.3f' % (v['events_per_s'], v['frac']))
"
BHIST_LIBRARY=$PWD/$lib timeout 300 python bench.py --config C3 --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline --secondary "" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('    C3 %.4g ev/s frac %.3f' % (d['value'], d['roofline']['frac']))"
done
