for c in C2 C1S C4W C3; do
ncu --set full --clock-control none --import-source on -k regex:k_fill -s 3 -c 1 -o gpurun_out/prof2_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu2_$c.log 2>&1
tail -1 gpurun_out/ncu2_$c.log
done
python bench.py --config C4W --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 | cut -c1-400
