ncu --set full --clock-control none --import-source on -k regex:k_fill_multi -s 2 -c 1 -o gpurun_out/prof6_C5 python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu6.log 2>&1
tail -1 gpurun_out/ncu6.log
