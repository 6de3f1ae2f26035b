#!/bin/bash
# Full GPU check: build+smoke, every gpu test, the default bench line, per-config rows.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests/ -q -m gpu --timeout=600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; cut -c1-400 gpurun_out/bench_default.json
rm -f gpurun_out/bench_cfgs.jsonl
for c in C1 C1S C3 C3W C4 C4W C5; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" >> gpurun_out/bench_cfgs.jsonl 2>>gpurun_out/bench_cfgs.err; done
timeout 300 python bench.py --config C3 --strategy sort --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" >> gpurun_out/bench_cfgs.jsonl 2>>gpurun_out/bench_cfgs.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1
