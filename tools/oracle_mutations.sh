#!/bin/bash
# Mutation check of the oracle pins (VERDICT r1 "done when"): each mutation of the oracle
# must turn the CPU suite (-m "not gpu") red; the file is restored after each one.
set -u
cd "$(dirname "$0")/.."
run() { python -c "import oracle; oracle.build(force=True)" >/dev/null 2>&1 || python -c "import oracle; oracle.build()" > /dev/null 2>&1; timeout 600 python -m pytest tests -m "not gpu" -x -q -p no:cacheprovider 2>&1 | tail -1; }
echo "== swap 9/10"; sed -i 's/add_stat(h, 9, (wi \* x\[0\]) \* x\[2\]);/add_stat(h, 9, (wi * x[1]) * x[2]);/; s/add_stat(h, 10, (wi \* x\[1\]) \* x\[2\]);/add_stat(h, 10, (wi * x[0]) * x[2]);/' oracle/bhist_oracle.c; git diff --stat oracle/; run; git checkout oracle/bhist_oracle.c
echo "== reciprocal"; sed -i 's|double q = ((double)nbins \* (x - xmin)) / (xmax - xmin);|double q = (x - xmin) * ((double)nbins / (xmax - xmin));|' oracle/bhist_oracle.c; git diff --stat oracle/; run; git checkout oracle/bhist_oracle.c
echo "== fmin->minimum"; sed -i 's/np.fmin(A, B)/np.minimum(A, B)/' oracle/expr.py; git diff --stat oracle/; run; git checkout oracle/expr.py
echo "== x/D*n"; sed -i 's|double q = ((double)nbins \* (x - xmin)) / (xmax - xmin);|double q = (double)nbins * ((x - xmin) / (xmax - xmin));|' oracle/bhist_oracle.c; git diff --stat oracle/; run; git checkout oracle/bhist_oracle.c
python -c "import oracle; oracle.build(force=True)" >/dev/null 2>&1 || true
