#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill -s 5 -c 1 -o gpurun_out/prof_small python tools/small_one.py 32768 2d > gpurun_out/ncu_small.log 2>&1
ls gpurun_out
