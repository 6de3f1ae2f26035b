#!/bin/bash
# A/B of two prebuilt libraries (A: build_ab/libbhist_A.so, B: the in-tree build) on the bench
# configs given as arguments; each line: [lib] ms_per_step frac (tools/gpu.sh envs job).
A=BHIST_LIBRARY=/root/repo/build_ab/libbhist_A.so
for c in "$@"; do echo "== $c"; bash tools/gpu.sh ab_run envs "$A;BHIST_LIBRARY=;$A;BHIST_LIBRARY=" --config $c; done
