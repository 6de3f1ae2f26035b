#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill -s 3 -c 1 -o gpurun_out/prof_c2new python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" > /dev/null 2>&1
BHIST_LIBRARY=$PWD/build_ab/libbhist_old.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill -s 3 -c 1 -o gpurun_out/prof_c2old python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" > /dev/null 2>&1
