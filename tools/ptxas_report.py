#!/usr/bin/env python
"""Compile csrc/bhist.cu with -Xptxas -v and print registers / spills per kernel."""
import re
import subprocess
import sys

import sys
src = sys.argv[1] if len(sys.argv) > 1 else "paper_2401_13310_b200/csrc/bhist.cu"
out = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xptxas", "-v",
                      "-I", "paper_2401_13310_b200/build/libbhist.so.obj", "-c", "-o", "/dev/null", src], capture_output=True, text=True).stderr
cur = None
rows = []
for line in out.splitlines():
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        cur = {"name": m.group(1)}
        rows.append(cur)
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        cur["spill"] = int(m.group(1)) + int(m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        cur["regs"] = int(m.group(1))
only_spill = "--spills" in sys.argv
for r in rows:
    if only_spill and not r.get("spill"):
        continue
    name = subprocess.run(["c++filt", r["name"]], capture_output=True, text=True).stdout.strip()
    print(f"{r.get('regs', '?'):>4} regs  {r.get('spill', 0):>5} B spill  {name[:110]}")
