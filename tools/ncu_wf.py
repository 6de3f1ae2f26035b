"""Per-SASS-instruction shared-memory wavefronts of one ncu --set full capture (source page):
   python tools/ncu_wf.py <report.ncu-rep> [events]  -> top instructions by L1 shared wavefronts."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
events = float(sys.argv[2]) if len(sys.argv) > 2 else 0
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
tot = inst = 0
out = []
for r in rows[2:]:
    try:
        wf = int(r[ix["L1 Wavefronts Shared"]])
        ideal = int(r[ix["L1 Wavefronts Shared Ideal"]])
        ex = int(r[ix["Instructions Executed"]])
        th = float(r[ix["Avg. Threads Executed"]])
        smp = int(r[ix["Warp Stall Sampling (All Samples)"]])
    except (ValueError, KeyError, IndexError):
        continue
    tot += wf
    inst += ex
    out.append((wf, ideal, ex, th, smp, r[1].strip()))
print(f"total shared wavefronts {tot:,}  warp instructions {inst:,}")
if events:
    print(f"per 32 events: wavefronts {32 * tot / events:.2f}  instructions {32 * inst / events:.1f}")
for o in sorted(out, reverse=True)[:16]:
    if o[0] == 0:
        break
    print("%11d ideal %11d exec %10d thr %4.1f wf/exec %5.2f  %s" % (o[0], o[1], o[2], o[3], o[0] / max(o[2], 1), o[5]))
smp_tot = sum(o[4] for o in out) or 1
print("top stall-sampled instructions:")
for o in sorted(out, key=lambda o: -o[4])[:12]:
    print("  %5.1f%%  %s" % (100.0 * o[4] / smp_tot, o[5]))
