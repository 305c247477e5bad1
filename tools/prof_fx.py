"""One fixed-point query batch (NEXT-1) for ncu: build the config's fx snapshot, run
v3db_query_batch_fx once (warm) + once (profiled region via cudaProfilerStart/Stop).
Usage: ncu --profile-from-start off ... python tools/prof_fx.py --config c4"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2603_03065_b200 import v3db  # noqa: E402
from synth import generate_float, get_config  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="c4")
p.add_argument("--trace", default="on")
args = p.parse_args()
cfg = get_config(args.config)
f = generate_float(cfg)
db = v3db.encode_fixed_point(torch.from_numpy(f.db).cuda(), f.v_max)
qs = v3db.encode_fixed_point(torch.from_numpy(f.queries).cuda(), f.v_max)
s = v3db.build_snapshot_fx(db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, f.centroid_rows, f.codeword_rows)
out = v3db.alloc_outputs_fx(s, cfg.Q, cfg.nprobe, cfg.k, trace=args.trace == "on")
v3db.query_batch_fx(s, qs, cfg.nprobe, cfg.k, out=out)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
v3db.query_batch_fx(s, qs, cfg.nprobe, cfg.k, out=out)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
