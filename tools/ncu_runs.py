#!/usr/bin/env python
"""Where a kernel's instructions go: runs of consecutive SASS instructions with equal execution
counts (straight-line blocks) from an ncu report's source page, largest first (in address order).

  python tools/ncu_runs.py gpurun_out/x.ncu-rep <kernel regex> [units (e.g. CTAs) to divide by] [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
units = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(j for j, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[h]
ie, src = hdr.index("Instructions Executed"), hdr.index("Source")
st = hdr.index("Warp Stall Sampling (All Samples)")
vals = []
for r in rows[h + 1:]:
    if len(r) > ie and r[0].startswith("0x"):
        vals.append((float(r[ie] or 0), int(r[0], 16), r[src], float(r[st] or 0)))
base = vals[0][1]
runs, cur = [], None
for v, a, s, smp in vals:
    if cur and abs(cur[0] - v) < 1:
        cur[2] += 1
        cur[3] = s
        cur[5] += smp
    else:
        if cur:
            runs.append(cur)
        cur = [v, a - base, 1, s, s, smp]
runs.append(cur)
tot = sum(v for v, *_ in vals)
tsmp = sum(r[5] for r in runs) or 1
print(f"total warp-instructions {tot:.0f} = {tot / units:.1f} per unit")
big = sorted(runs, key=lambda r: -r[0] * r[2])[:top]
for r in sorted(big, key=lambda r: r[1]):
    print(f"{r[1]:6x} n={r[2]:4d} x{r[0] / units:8.1f} = {r[0] * r[2] / tot * 100:5.1f}% inst {r[5] / tsmp * 100:5.1f}% stall"
          f"  {r[4][:38]} .. {r[3][:38]}")
