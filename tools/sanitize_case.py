"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck): builds tiny
snapshots and runs both scan kernels, the W32 and P64 geometries and the mma.sync coarse path.
Checks results against the oracle so a sanitizer run is also a parity run."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2603_03065_b200 import v3db  # noqa: E402
from synth import generate, get_config  # noqa: E402

for name, nq in (("c0", 64), ("e2_basic", 40), ("c4_mini", 24), ("e2_large", 16)):
    cfg = get_config(name)
    inp = generate(cfg)
    ref_s = oracle.build_snapshot(inp.db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    qs = np.ascontiguousarray(inp.queries[:nq])
    ref = oracle.query_batch(ref_s, qs, cfg.nprobe, cfg.k)
    for mode in ("", "w32"):
        if mode:
            os.environ["V3DB_LUT_MODE"] = mode
        else:
            os.environ.pop("V3DB_LUT_MODE", None)
        s = v3db.build_snapshot(torch.from_numpy(inp.db).cuda(), cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows,
                                inp.codeword_rows)
        for algo in (1, 0):
            out = v3db.query_batch(s, torch.from_numpy(qs).cuda(), cfg.nprobe, cfg.k, algo=algo)
            torch.cuda.synchronize()
            for key, exp in ref.items():
                assert np.array_equal(out[key].cpu().numpy(), exp), (name, mode, algo, key)
        s.free()
    print("ok", name, flush=True)
