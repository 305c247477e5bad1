#!/usr/bin/env python
"""Warp-stall samples of one kernel aggregated by CUDA source line (ncu source page, cuda,sass view).

  python tools/ncu_lines.py gpurun_out/x.ncu-rep <kernel regex> [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(r for r in rows if r and r[0] == "Line No")
i_s = h.index("Warp Stall Sampling (All Samples)")
i_n = h.index("Instructions Executed")
stalls = [j for j, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
agg = collections.defaultdict(lambda: [0, 0, collections.Counter(), ""])
line, src, fname = None, "", ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) < len(h) or r[0] == "Line No":
        continue
    if r[0]:
        line, src = f"{fname}:{r[0]}", r[1].strip()
        continue
    if line is None:
        continue
    try:
        s, n = int(r[i_s] or 0), int(r[i_n] or 0)
    except ValueError:
        continue
    a = agg[line]
    a[0] += s
    a[1] += n
    a[3] = src
    for j in stalls:
        if r[j]:
            a[2][h[j][6:]] += int(r[j])
tot = sum(v[0] for v in agg.values()) or 1
print(f"total samples {tot}")
for ln, (s, n, st, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    main = ", ".join(f"{k}:{v}" for k, v in st.most_common(2))
    print(f"{100 * s / tot:5.1f}% {n:>10} {ln:<16} {src[:70]:<70} {main}")
