"""Time v3db_witness_batch (the prover witness of challenged queries) on a config, CUDA events."""
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
p.add_argument("--nq", type=int, default=1)
args = p.parse_args()
cfg = get_config(args.config)
inp = generate(cfg)
s = v3db.build_snapshot(torch.from_numpy(inp.db).cuda(), cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows,
                        inp.codeword_rows)
q = torch.from_numpy(inp.queries[:args.nq]).cuda().contiguous()
v3db.witness_batch(s, q, cfg.nprobe)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    w = v3db.witness_batch(s, q, cfg.nprobe)
b.record()
torch.cuda.synchronize()
mb = sum(t.numel() * 4 for t in w.values()) / 1e6
print(f"{cfg.name} witness nq={args.nq}: {a.elapsed_time(b) / 5:.3f} ms per batch, {mb:.1f} MB of witness")
