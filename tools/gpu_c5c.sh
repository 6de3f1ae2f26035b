for t in 512 768 1024; do for a in 0 1; do
echo "threads=$t agg_unit=$a"
BHIST_MULTI_THREADS=$t BHIST_MULTI_AGG_UNIT=$a ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_fill_multi --csv python bench.py --config C5 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>/dev/null | grep k_fill_multi | tail -1 | awk -F'","' '{print $NF}'
done; done
BHIST_MULTI_THREADS=768 timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -m "gpu" -k "multi or C5" 2>&1 | tail -2
BHIST_MULTI_AGG_UNIT=0 timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -m "gpu" -k "multi or C5" 2>&1 | tail -2
