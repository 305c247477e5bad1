"""Per-CTA start / end times of lm_kernel (experiment build -DLM_EXP_TIMES=1, tools/exp_build.sh):
how much of the kernel is a tail of a few late CTAs.

  tools/exp_build.sh times -DLM_EXP_TIMES=1
  V3DB_LIB=$PWD/exp/libv3db_times.so python tools/lm_times.py --config c4
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_03065_b200 import _lib, v3db  # noqa: E402
from synth import generate, get_config  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="c4")
args = p.parse_args()
cfg = get_config(args.config)
inp = generate(cfg)
db = torch.from_numpy(inp.db).cuda()
s = v3db.build_snapshot(db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
q = torch.from_numpy(inp.queries).cuda()
out = v3db.alloc_outputs(s, cfg.Q, cfg.nprobe, cfg.k, trace=True, device="cuda")
lib = _lib.load()
buf = (ctypes.c_ulonglong * 512)()
for rep in range(3):
    v3db.query_batch(s, q, cfg.nprobe, cfg.k, out=out)
    torch.cuda.synchronize()
    assert lib.v3db_exp_lm_times(buf) == 0
    t = np.array(buf[:], dtype=np.int64).reshape(256, 2)
    t = t[t[:, 1] > 0]
    t0 = t[:, 0].min()
    end = (t[:, 1] - t0) / 1e3
    print(f"{cfg.name} rep {rep}: {len(t)} CTAs, kernel {end.max():.1f} us; CTA end mean {end.mean():.1f} "
          f"median {np.median(end):.1f} min {end.min():.1f} us; mean/max {end.mean() / end.max():.3f}; "
          f"start spread {(t[:, 0].max() - t0) / 1e3:.1f} us")
