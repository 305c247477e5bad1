"""Time query_batch on a config with CUDA events (per-kernel via the profiling hooks)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2603_03065_b200 import v3db  # noqa: E402
from synth import generate, get_config  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="c4")
p.add_argument("--reps", type=int, default=5)
p.add_argument("--algos", default="1,2")
p.add_argument("--Q", type=int, default=0, help="use only the first Q queries")
p.add_argument("--k", type=int, default=0, help="override k")
p.add_argument("--nprobe", type=int, default=0, help="override nprobe")
p.add_argument("--trace", default="on")
p.add_argument("--opts", default="", help="comma-separated runs after the plain run, each OPT=VALUE[:OPT=VALUE] "
               "(v3db.OPT_* names without the prefix, e.g. SCAN_SEG=8:SCAN_NS=4)")
args = p.parse_args()
cfg = get_config(args.config)
inp = generate(cfg)
s = v3db.build_snapshot(torch.from_numpy(inp.db).cuda(), cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows,
                        inp.codeword_rows)
q = torch.from_numpy(inp.queries[: args.Q or None]).cuda().contiguous()
if args.Q:
    cfg = cfg.with_(Q=args.Q)
if args.k:
    cfg = cfg.with_(k=args.k)
if args.nprobe:
    cfg = cfg.with_(nprobe=args.nprobe)
out = v3db.alloc_outputs(s, cfg.Q, cfg.nprobe, cfg.k, trace=args.trace == "on", device="cuda")
v3db.profile_enable(True)
for env in [""] + [e for e in args.opts.split(",") if e]:
    for kv in env.split(":"):
        if kv:
            k, v = kv.split("=")
            v3db.set_option(getattr(v3db, "OPT_" + k), int(v))
    for algo in [int(x) for x in args.algos.split(",")]:
        v3db.query_batch(s, q, cfg.nprobe, cfg.k, out=out, algo=algo)
        ts = []
        for _ in range(args.reps):
            v3db.query_batch(s, q, cfg.nprobe, cfg.k, out=out, algo=algo)
            ts.append(v3db.profile_read(detail=True))
        med = [sorted(t[i] for t in ts)[len(ts) // 2] for i in range(5)]
        print(f"{cfg.name} opts={env or '-'} algo={algo} coarse {med[0]:.3f} ms  scan {med[1]:.3f} ms "
              f"(prologue {med[3]:.3f}, main {med[2]:.3f}, select {med[4]:.3f})", flush=True)
