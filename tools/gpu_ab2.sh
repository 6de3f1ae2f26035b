for lib in paper_2401_13310_b200/libbhist.so build_ab/libbhist_NOCAS.so build_ab/libbhist_NOSEARCH.so build_ab/libbhist_both.so; do
BHIST_LIBRARY=$PWD/$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$lib C2 %.4g ev/s frac %.3f'%(d['value'], d['roofline']['frac']))"; done
