for c in C2 C1S; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill -s 3 -c 1 -o gpurun_out/prof12_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu12_$c.log 2>&1
done
