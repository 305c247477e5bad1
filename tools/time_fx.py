"""NEXT-1 measurement: the 16-bit fixed-point path per config -- GPU encoding,
build time, and the query batch (Steps 1-2 / Steps 3-5 split via the profile hooks), trace on/off.
Queries/s = nq / device time of one v3db_query_batch_fx call (CUDA events, L2 flushed between
runs).  Usage: python tools/time_fx.py --configs c1,c2 [--reps 5]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2603_03065_b200 import v3db  # noqa: E402
from synth import generate_float, get_config  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--configs", default="c1,c2")
p.add_argument("--reps", type=int, default=5)
p.add_argument("--opts", default="", help="OPT=VALUE[:OPT=VALUE] set before the runs (v3db.OPT_* names without the prefix)")
args = p.parse_args()
for kv in args.opts.split(":"):
    if kv:
        k, v = kv.split("=")
        v3db.set_option(getattr(v3db, "OPT_" + k), int(v))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name in args.configs.split(","):
    cfg = get_config(name)
    f = generate_float(cfg)
    xdb = torch.from_numpy(f.db).cuda()
    xq = torch.from_numpy(f.queries).cuda()
    db = v3db.encode_fixed_point(xdb, f.v_max)
    qs = v3db.encode_fixed_point(xq, f.v_max)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = v3db.build_snapshot_fx(db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, f.centroid_rows, f.codeword_rows)
    build_s = time.perf_counter() - t0
    res = {"config": name, "build_s": round(build_s, 3)}
    for trace in (True, False):
        v3db.query_batch_fx(s, qs, cfg.nprobe, cfg.k, trace=trace)
        ms, coarse, scan = [], [], []
        v3db.profile_enable(True)
        for _ in range(args.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            v3db.query_batch_fx(s, qs, cfg.nprobe, cfg.k, trace=trace)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
            c, sc = v3db.profile_read()
            coarse.append(c)
            scan.append(sc)
        v3db.profile_enable(False)
        ms.sort()
        med = ms[len(ms) // 2]
        tag = "trace" if trace else "notrace"
        res[f"ms_{tag}"] = round(med, 3)
        res[f"qps_{tag}"] = round(cfg.Q / med * 1e3)
        res[f"coarse_ms_{tag}"] = round(sorted(coarse)[len(coarse) // 2], 3)
        res[f"scan_ms_{tag}"] = round(sorted(scan)[len(scan) // 2], 3)
    s.free()
    print(json.dumps(res), flush=True)
