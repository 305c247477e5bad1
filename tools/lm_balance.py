"""Load balance of lm_kernel's static round-robin over the work items (diagnostic, GPU box).

Rebuilds the item list of a config from the query's probe lists (trace_lists) and the snapshot's
counts, charges each item  tiles(cnt) x chunk-rounds(np)  (the epilogue's unit of work per warp),
and prints max / mean of the per-CTA sums for the round-robin deal and for a cost-sorted deal.

  python tools/lm_balance.py --config c4
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_03065_b200 import v3db  # noqa: E402
from synth import generate, get_config  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="c4")
p.add_argument("--nt", type=int, default=64)
p.add_argument("--ctas", type=int, default=148)
args = p.parse_args()
cfg = get_config(args.config)
inp = generate(cfg)
db = torch.from_numpy(inp.db).cuda()
s = v3db.build_snapshot(db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
q = torch.from_numpy(inp.queries).cuda()
out = v3db.query_batch(s, q, cfg.nprobe, cfg.k, trace=True)
torch.cuda.synchronize()
lists = out["trace_lists"].cpu().numpy().ravel()
counts = v3db.snapshot_export(s, v3db.FIELD_COUNTS).astype(np.int64)
h = np.bincount(lists, minlength=cfg.nlist)
NT = args.nt
cost, pairs = [], []
for i in range(cfg.nlist):
    tiles = (counts[i] + 127) // 128
    pad_tiles = (cfg.L + 127) // 128 - tiles
    for o in range(0, h[i], NT):
        n = min(NT, h[i] - o)
        rounds = (((n + 15) // 16) + 1) // 2
        cost.append(tiles * rounds + 0.25 * pad_tiles * rounds + 0.5)
        pairs.append(n)
cost = np.array(cost)
print(f"{cfg.name}: {len(cost)} items, pairs/list mean {h.mean():.1f} max {h.max()}, item pairs mean {np.mean(pairs):.1f}")


def deal(order):
    per = np.zeros(args.ctas)
    for r, j in enumerate(order):
        per[r % args.ctas] += cost[j]
    return per


for name, order in (("list order (current)", np.arange(len(cost))),
                    ("cost-sorted descending", np.argsort(-cost, kind="stable"))):
    per = deal(order)
    print(f"  {name:<26} max/mean {per.max() / per.mean():.4f}  min/mean {per.min() / per.mean():.4f}")
# greedy LPT as the bound
per = np.zeros(args.ctas)
for j in np.argsort(-cost, kind="stable"):
    per[per.argmin()] += cost[j]
print(f"  {'LPT (bound)':<26} max/mean {per.max() / per.mean():.4f}")
