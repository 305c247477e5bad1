#!/usr/bin/env python
"""Summarise ncu captures for profiles/: key metrics of every kernel in a .ncu-rep (raw
page) and the per-kernel share of a launch list CSV (gpu__time_duration.sum).

  python tools/ncu_summary.py rep  gpurun_out/prof.ncu-rep   > profiles/x.md
  python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/y.md
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size",
    "sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active",
    "sm__cycles_elapsed.avg.per_second", "smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct",
    "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct",
    "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    # tensor pipe (tcgen05 kind::i8: the coarse kernels)
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum",
]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    print(f"# ncu --set full summary: `{path.split('/')[-1]}`\n")
    for v in rows[2:]:
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"## {name[:140]}\n\n| metric | value | unit |\n|---|---|---|")
        for k in KEYS:  # raw column names may carry a section prefix ("TPC.TriageCompute.")
            i = next((j for j, col in enumerate(h) if col == k or col.endswith("." + k)), None)
            if i is not None and v[i] not in ("", "n/a"):
                print(f"| {k} | {v[i]} | {units[i]} |")
        print()


def launches(path):
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        name = r[ki].split("(")[0]
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(r[ui], 1e-6)
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values())
    print(f"# launch list `{path.split('/')[-1]}` (ncu gpu__time_duration.sum, cold-cache, serialised)\n")
    print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for name, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{name[:110]}` | {n} | {ms:.3f} | {100 * ms / tot:.1f}% |")


if __name__ == "__main__":
    {"rep": rep, "launches": launches}[sys.argv[1]](sys.argv[2])
