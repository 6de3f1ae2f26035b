#!/bin/bash
# One ncu --set full capture of the dominant fill kernel per config; summaries only come back.
mkdir -p gpurun_out
prof() {  # name, kernel regex, skip, bench args...
  local name=$1 kre=$2 skip=$3; shift 3
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s $skip -c 1 -o /tmp/prof_$name \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" "$@" > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/prof_$name.ncu-rep > gpurun_out/ncu_v8_$name.txt 2>&1
  python tools/ncu_opmix.py /tmp/prof_$name.ncu-rep "regex:$kre" >> gpurun_out/ncu_v8_$name.txt 2>&1
  rm -f /tmp/prof_$name.ncu-rep
}
prof C1S k_fill 3 --config C1S
prof C3_sort_pass1 k_part_scatter 3 --config C3
prof C3W k_fill 3 --config C3W
prof C4 k_fill 3 --config C4
prof C4W k_fill 3 --config C4W
prof C5_H7 k_fill 31 --config C5
timeout 1200 python -m pytest tests/test_parity_gpu.py -q -m gpu -x -k "bench_json or bench_two" > gpurun_out/pytest_bench.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_bench.log
ls gpurun_out
