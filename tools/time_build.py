"""Snapshot build time per shaping rule (BASELINE.json greedy vs the paper's Alg. 1) and Alg. 1's
moved-vector count / rounds (the paper reports "moved" next to train time)."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_03065_b200 import v3db  # noqa: E402
from synth import generate, get_config  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--configs", default="c1,c2,c3,c4")
args = p.parse_args()
for name in args.configs.split(","):
    cfg = get_config(name)
    inp = generate(cfg)
    db = torch.from_numpy(inp.db).cuda()
    for rule, rname in ((v3db.SHAPE_GREEDY, "greedy"), (v3db.SHAPE_REBALANCE, "alg1")):
        v3db.build_snapshot(db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows, rule=rule).free()
        torch.cuda.synchronize()
        st = {}
        t0 = time.perf_counter()
        s = v3db.build_snapshot(db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows, rule=rule,
                                stats=st)
        dt = time.perf_counter() - t0
        counts = v3db.snapshot_export(s, v3db.FIELD_COUNTS)
        s.free()
        print(f"{name} {rname}: build {dt:.3f} s, moved {st['moved']}, rounds {st['rounds']}, "
              f"full lists {int((counts == cfg.L).sum())}/{cfg.nlist}", flush=True)
