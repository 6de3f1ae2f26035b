for solo in 0 1; do
BHIST_MULTI_SOLO=$solo timeout 300 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('solo=$solo C5 %.4g ev/s ms %.3f'%(d['value'], d['ms_per_step']))"
done
BHIST_MULTI_SOLO=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5e.csv python bench.py --config C5 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
