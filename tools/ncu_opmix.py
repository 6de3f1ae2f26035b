"""Executed-instruction mix by SASS opcode for one kernel of an .ncu-rep."""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", kern],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = [r for r in csv.DictReader(io.StringIO("\n".join(lines[start:]))) if r["Address"].startswith("0x")]
seen = set()
mix = collections.Counter()
for r in rows:
    if r["Address"] in seen:
        continue
    seen.add(r["Address"])
    src = r["Source"].strip()
    op = src.split()[1] if src.startswith("@") else src.split()[0]
    mix[op.split(".")[0]] += int(r["Instructions Executed"] or 0)
tot = sum(mix.values())
print(f"{kern}: {tot} warp instructions")
for op, c in mix.most_common(30):
    print(f"{op:12s} {c:12d} {100*c/tot:5.1f}%")
