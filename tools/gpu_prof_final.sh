#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --secondary "" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill -s 3 -c 1 -o /tmp/prof_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" > /dev/null 2>&1
python tools/ncu_summary.py /tmp/prof_c2.ncu-rep > gpurun_out/ncu_v10_C2.txt 2>&1; python tools/ncu_opmix.py /tmp/prof_c2.ncu-rep regex:k_fill >> gpurun_out/ncu_v10_C2.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_part -s 3 -c 3 -o /tmp/prof_c3 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" > /dev/null 2>&1
python tools/ncu_summary.py /tmp/prof_c3.ncu-rep > gpurun_out/ncu_v10_C3_sort.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_C3.csv python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" > /dev/null 2>&1
