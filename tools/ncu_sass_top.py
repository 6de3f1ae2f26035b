"""Top stall-sampled SASS lines of one kernel in an .ncu-rep (ncu -i --page source --print-source sass)."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", kern],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = [r for r in csv.DictReader(io.StringIO("\n".join(lines[start:]))) if r["Address"].startswith("0x")]
tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
rows.sort(key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))
print(f"{kern}: {tot} samples, {len(rows)} SASS lines")
for r in rows[:top]:
    s = int(r["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{100*s/tot:5.1f}%  {r['Address'][-5:]}  {r['Source'].strip()[:90]}")
