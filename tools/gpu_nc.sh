#!/bin/bash
mkdir -p gpurun_out
BHIST_LIBRARY=$PWD/build_ab/libbhist_nc.so timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_part_scatter" -s 3 -c 1 -o /tmp/nc python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" > /dev/null 2>&1
python tools/ncu_summary.py /tmp/nc.ncu-rep > gpurun_out/nc.txt 2>&1; python tools/ncu_opmix.py /tmp/nc.ncu-rep regex:k_part_scatter >> gpurun_out/nc.txt 2>&1
python tools/ncu_sass_top.py /tmp/nc.ncu-rep regex:k_part_scatter 20 >> gpurun_out/nc.txt 2>&1
