#!/bin/bash
# Round profiling recipe (run under gpurun): launch list of the default bench command and
# one ncu --set full capture of the top kernel; summaries are copied to profiles/ by hand.
set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_default.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline \
    > gpurun_out/launches_default.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fill -s 3 -c 1 \
    -o gpurun_out/prof_default python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
    > gpurun_out/prof_default.log 2>&1
