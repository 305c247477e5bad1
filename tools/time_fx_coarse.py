"""Experiment timing of the fixed-point Steps 1-2 alone (profile hook 'coarse'): the snapshot is built
with the FP64 kernel (OPT_FX_COARSE=1), the query batch runs the default path.  Usage (under gpurun):
V3DB_LIB=path.so python tools/time_fx_coarse.py --config c4"""
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
p.add_argument("--reps", type=int, default=5)
args = p.parse_args()
cfg = get_config(args.config)
f = generate_float(cfg)
db = v3db.encode_fixed_point(torch.from_numpy(f.db).cuda(), f.v_max)
qs = v3db.encode_fixed_point(torch.from_numpy(f.queries).cuda(), f.v_max)
with v3db.option(v3db.OPT_FX_COARSE, 1):
    s = v3db.build_snapshot_fx(db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, f.centroid_rows, f.codeword_rows)
v3db.query_batch_fx(s, qs, cfg.nprobe, cfg.k, trace=False)
v3db.profile_enable(True)
cs = []
for _ in range(args.reps):
    v3db.query_batch_fx(s, qs, cfg.nprobe, cfg.k, trace=False)
    cs.append(v3db.profile_read()[0])
print(os.environ.get("V3DB_LIB", "default"), cfg.name, "coarse ms", sorted(cs)[len(cs) // 2], flush=True)
