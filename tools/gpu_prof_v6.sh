#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_C5.csv python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --secondary "" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill -s 3 -c 1 -o gpurun_out/prof_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill -s 27 -c 8 -o gpurun_out/prof_c5 python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" > /dev/null 2>&1
ls -la gpurun_out
