#!/usr/bin/env python
"""Hot SASS instructions of one kernel in an ncu report (source page): the top instructions by
warp-stall samples and by instructions executed, with the dominant stall reasons.

  python tools/ncu_hot.py gpurun_out/x.ncu-rep <kernel regex> [top] [launch skip]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
skip = ["--launch-skip", sys.argv[4], "--launch-count", "1"] if len(sys.argv) > 4 else []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", *skip],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, ln in enumerate(lines) if ln.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
ix = {k: h.index(k) for k in h}
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
data = []
for r in rows[1:]:
    if len(r) < len(h):
        continue
    try:
        data.append((int(r[ix["Warp Stall Sampling (All Samples)"]] or 0), int(r[ix["Instructions Executed"]] or 0),
                     r[ix["Address"]][-5:], r[ix["Source"]].strip(), {k: int(r[ix[k]] or 0) for k in stalls}))
    except ValueError:
        continue
tot_s = sum(d[0] for d in data) or 1
tot_i = sum(d[1] for d in data) or 1
print(f"total samples {tot_s}, instructions {tot_i}")
agg = {k: sum(d[4][k] for d in data) for k in stalls}
print("stalls:", ", ".join(f"{k[6:]} {100 * v / tot_s:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
print(f"\n-- top {top} by stall samples (in address order)")
sel = sorted(sorted(data, key=lambda d: -d[0])[:top], key=lambda d: d[2])
for s, n, a, src, st in sel:
    main = ", ".join(f"{k[6:]}:{v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:2] if v)
    print(f"{a} {100 * s / tot_s:5.1f}% {n:>11} {src[:70]:70s} {main}")
