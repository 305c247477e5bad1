"""Recall@k of the fixed-shape IVF-PQ query path against exact k-NN on the same synthetic data
(SURVEY.md §8(c) "Paper numbers": a plausibility check only -- the paper reports zk recall ~ the
standard IVF-PQ's on SIFT1M / GIST1M / MS MARCO, datasets not available here).

  python tools/recall.py [--config c1] [--out profiles/recall_r02.json]

int8: BASELINE.json's int8 vectors, exact squared L2 over them.  fx16: the paper's 16-bit fixed
point encoding of the same float draws, exact squared L2 over the encoded
vectors.  Exact k-NN runs on the GPU with torch (float64 for fx16, float32 exact below 2^24 for
int8), ties broken by the lower id like Step 5 (R10).  Recall@k = |IVF-PQ top-k & exact top-k| / k.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2603_03065_b200 import v3db  # noqa: E402
from synth import generate, generate_float, get_config  # noqa: E402


def exact_topk(db: torch.Tensor, q: torch.Tensor, k: int, dtype) -> np.ndarray:
    """Exact k nearest ids by (squared L2, id), chunked over queries."""
    dbf = db.to(dtype)
    dn = (dbf * dbf).sum(1)
    out = []
    for lo in range(0, q.shape[0], 1024):
        qf = q[lo:lo + 1024].to(dtype)
        d = (qf * qf).sum(1, keepdim=True) + dn[None, :] - 2.0 * qf @ dbf.T
        # (d, id) order: a stable sort by d keeps ascending ids among ties
        idx = torch.sort(d, dim=1, stable=True).indices[:, :k]
        out.append(idx.cpu().numpy())
    return np.concatenate(out)


def recall(got: np.ndarray, exp: np.ndarray, k: int) -> float:
    hits = [len(np.intersect1d(g[:k], e[:k])) for g, e in zip(got, exp)]
    return float(np.mean(hits)) / k


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c1")
    p.add_argument("--out", default="")
    args = p.parse_args()
    cfg = get_config(args.config)
    K = 100
    res = {"config": cfg.name, "Q": cfg.Q, "N": cfg.N, "nlist": cfg.nlist, "L": cfg.L, "M": cfg.M, "Ks": cfg.Ks,
           "nprobe": cfg.nprobe, "data": "synthetic (synth/generate.py)", "exact": "brute-force squared L2, torch"}
    inp = generate(cfg)
    db = torch.from_numpy(inp.db).cuda()
    q = torch.from_numpy(inp.queries).cuda()
    s = v3db.build_snapshot(db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    exp = exact_topk(db, q, K, torch.float32)
    res["int8"] = {}
    for nprobe in sorted({cfg.nprobe, 2 * cfg.nprobe, 4 * cfg.nprobe}):
        if nprobe > cfg.nlist:
            continue
        out = v3db.query_batch(s, q, nprobe, K, trace=False)
        got = out["out_ids"].cpu().numpy()
        res["int8"][f"nprobe={nprobe}"] = {"recall@1": recall(got, exp, 1), "recall@10": recall(got, exp, 10),
                                           "recall@100": recall(got, exp, 100)}
    s.free()
    f = generate_float(cfg)
    fdb = v3db.encode_fixed_point(torch.from_numpy(f.db).cuda(), f.v_max)
    fq = v3db.encode_fixed_point(torch.from_numpy(f.queries).cuda(), f.v_max)
    sf = v3db.build_snapshot_fx(fdb, cfg.nlist, cfg.L, cfg.M, cfg.Ks, f.centroid_rows, f.codeword_rows)
    expf = exact_topk(fdb, fq, K, torch.float64)
    res["fx16"] = {}
    for nprobe in sorted({cfg.nprobe, 2 * cfg.nprobe, 4 * cfg.nprobe}):
        if nprobe > cfg.nlist:
            continue
        out = v3db.query_batch_fx(sf, fq, nprobe, K, trace=False)
        got = out["out_ids"].cpu().numpy()
        res["fx16"][f"nprobe={nprobe}"] = {"recall@1": recall(got, expf, 1), "recall@10": recall(got, expf, 10),
                                           "recall@100": recall(got, expf, 100)}
    sf.free()
    line = json.dumps(res)
    print(line)
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
