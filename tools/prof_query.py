"""Profiling driver: build a config's snapshot, then run `--reps` query batches inside
cudaProfilerStart/Stop so `ncu --profile-from-start off` sees only the query path.

  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv python tools/prof_query.py --config c4
"""
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
p.add_argument("--reps", type=int, default=2)
p.add_argument("--algo", type=int, default=0)
p.add_argument("--trace", default="on")
args = p.parse_args()
cfg = get_config(args.config)
inp = generate(cfg)
db = torch.from_numpy(inp.db).cuda()
s = v3db.build_snapshot(db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
del db
q = torch.from_numpy(inp.queries).cuda()
out = v3db.alloc_outputs(s, cfg.Q, cfg.nprobe, cfg.k, trace=args.trace == "on", device="cuda")
v3db.query_batch(s, q, cfg.nprobe, cfg.k, out=out, algo=args.algo)   # warm-up (pool, attributes)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(args.reps):
    v3db.query_batch(s, q, cfg.nprobe, cfg.k, out=out, algo=args.algo)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok", cfg.name)
