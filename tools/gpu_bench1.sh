set -x
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c2.jsonl 2> gpurun_out/bench_c2.err; tail -3 gpurun_out/bench_c2.err
cat gpurun_out/bench_c2.jsonl
for c in C1S C1 C3 C3W C4 C4W; do python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 >> gpurun_out/bench_cfgs.jsonl 2>>gpurun_out/bench_cfgs.err; done
cat gpurun_out/bench_cfgs.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config']['workload'][:40], d['config']['fill_strategy'], '%.3g ev/s'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'launch_ms %.3f'%d['roofline']['launch_ms'], 'e2e %.3g'%d['e2e']['value'], d['clocks'])
"
tail -3 gpurun_out/bench_cfgs.err
python bench.py --impl reference --steps 3 --warmup 3
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fill -s 3 -c 1 -o gpurun_out/prof_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_c2.log 2>&1
tail -2 gpurun_out/ncu_c2.log
