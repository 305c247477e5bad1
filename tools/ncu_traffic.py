#!/usr/bin/env python
"""DRAM bytes (read + write) per launch of one kernel in an ncu report: prints `<report> <kernel> <bytes>`.
  python tools/ncu_traffic.py gpurun_out/x.ncu-rep lm_kernel"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", f"regex:{kern}",
                      "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(i for i, r in enumerate(rows) if "dram__bytes_read.sum" in r)
hdr, units = rows[h], rows[h + 1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for r in rows[h + 2:h + 3]:
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        j = hdr.index(m)
        tot += float(r[j].replace(",", "")) * scale.get(units[j], 1)
    print(rep, kern, int(tot))
