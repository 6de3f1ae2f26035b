#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu --timeout=300 -x -k "fill_parity or tiny or peaked or multi or exact or expr" > gpurun_out/pytest_s.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_s.log
python tools/small_fill.py
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_small.csv python tools/small_fill.py > /dev/null 2>&1
python - <<'PY'
import csv
lines=open("gpurun_out/launch_small.csv").read().splitlines()
i=next(k for k,l in enumerate(lines) if l.startswith('"ID"'))
rows=list(csv.DictReader(lines[i:]))
import collections
d=collections.defaultdict(list)
for r in rows: d[(r["Kernel Name"][:40], r["Grid Size"])].append(float(r["Metric Value"].replace(',','')))
for k,v in d.items(): print(k, len(v), "median %.2f us"%(sorted(v)[len(v)//2]/1e3))
PY
