#!/bin/bash
mkdir -p gpurun_out
for c in C3 C4W; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:k_part -c 9 --log-file gpurun_out/sort_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" --strategy sort > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_part -s 3 -c 3 -o gpurun_out/prof_sort_C3 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" > /dev/null 2>&1
ls -la gpurun_out
