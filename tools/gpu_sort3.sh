#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu --timeout=300 -x -k "sort" > gpurun_out/pytest_sort.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_sort.log
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" "$@" 2>>gpurun_out/sort.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config']['workload'][:12], d['config']['fill_strategy'][:12], '%.4g ev/s'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'launch_ms %.3f'%d['roofline']['launch_ms'], 'ms/step %.3f'%d['ms_per_step'], 'e2e %.3g'%d['e2e']['value'])
"; }
for c in C3 C3W C4; do run --config $c --strategy sort; done
run --config C1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k_part -c 6 --log-file gpurun_out/sort_C3.csv python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" --strategy sort > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_part_scatter -s 1 -c 1 -o gpurun_out/prof_sort_C3 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" --strategy sort > /dev/null 2>&1
