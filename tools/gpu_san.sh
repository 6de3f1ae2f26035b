#!/bin/bash
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  echo "== $tool"; timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py 2>&1 | grep -v "^frame" | tail -6
done
