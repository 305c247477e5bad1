"""Small end-to-end workload for the debug library (V3DB_LIB=debug: device-side invariant traps
on every shared-memory append / stage write, V3DB_SYNC_CHECK=1 launch checks) and for
compute-sanitizer where it is available.  Builds tiny snapshots and runs every scan kernel, the
W32 and P64 geometries, the mma.sync coarse path and the fixed-point path; checks results against
the oracle so a checked run is also a parity run.  Exit code 0 = every case matched."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2603_03065_b200 import v3db  # noqa: E402
from synth import generate, generate_float, get_config  # noqa: E402

names = sys.argv[1:] or ["c0", "e2_basic", "c4_mini", "e2_large"]
nq_of = {"c0": 64, "e2_basic": 40, "c4_mini": 24, "e2_large": 16}
algos = [v3db.SCAN_GENERIC, v3db.SCAN_ROTATED] + ([v3db.SCAN_LIST_MAJOR] if hasattr(v3db, "SCAN_LIST_MAJOR") else [])
for name in names:
    cfg = get_config(name)
    nq = nq_of.get(name, 32)
    inp = generate(cfg)
    ref_s = oracle.build_snapshot(inp.db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    qs = np.ascontiguousarray(inp.queries[:nq])
    ref = oracle.query_batch(ref_s, qs, cfg.nprobe, cfg.k)
    for mode in (0, 1):
        v3db.set_option(v3db.OPT_LUT_W32, mode)
        s = v3db.build_snapshot(torch.from_numpy(inp.db).cuda(), cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows,
                                inp.codeword_rows)
        for algo in algos:
            try:
                out = v3db.query_batch(s, torch.from_numpy(qs).cuda(), cfg.nprobe, cfg.k, algo=algo)
            except v3db.V3DBError as exc:   # a kernel this shape does not support (EINVAL)
                assert exc.status == 1, exc
                continue
            torch.cuda.synchronize()
            for key, exp in ref.items():
                assert np.array_equal(out[key].cpu().numpy(), exp), (name, mode, algo, key)
        s.free()
    v3db.set_option(v3db.OPT_LUT_W32, 0)
    # the other exact paths of the default (list-major) query: CTA / warp Step 5, 4 keys per coarse block,
    # the group-minimum coarse passes
    for opt_key, val in ((v3db.OPT_SELECT_CTA, 1), (v3db.OPT_SELECT_CTA, 2), (v3db.OPT_COARSE_KEYS, 4),
                         (v3db.OPT_COARSE_2PASS, 1), (v3db.OPT_COARSE_2PASS, 8)):
        with v3db.option(opt_key, val):
            s = v3db.build_snapshot(torch.from_numpy(inp.db).cuda(), cfg.nlist, cfg.L, cfg.M, cfg.Ks,
                                    inp.centroid_rows, inp.codeword_rows)
            out = v3db.query_batch(s, torch.from_numpy(qs).cuda(), cfg.nprobe, cfg.k)
            torch.cuda.synchronize()
            for key, exp in ref.items():
                assert np.array_equal(out[key].cpu().numpy(), exp), (name, opt_key, val, key)
            s.free()
    with v3db.option(v3db.OPT_COARSE_SIMT, 1):
        s = v3db.build_snapshot(torch.from_numpy(inp.db).cuda(), cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows,
                                inp.codeword_rows)
        out = v3db.query_batch(s, torch.from_numpy(qs).cuda(), cfg.nprobe, cfg.k)
        torch.cuda.synchronize()
        for key, exp in ref.items():
            assert np.array_equal(out[key].cpu().numpy(), exp), (name, "simt", key)
        s.free()
    # NEXT-1 fixed point on the same shape
    f = generate_float(cfg)
    fdb = oracle.encode_fixed_point(f.db, f.v_max)
    fq = np.ascontiguousarray(oracle.encode_fixed_point(f.queries[:nq], f.v_max))
    ref_f = oracle.build_snapshot(fdb, cfg.nlist, cfg.L, cfg.M, cfg.Ks, f.centroid_rows, f.codeword_rows)
    reff = oracle.query_batch(ref_f, fq, cfg.nprobe, cfg.k)
    # (tensor-core coarse + list-major scan by default; then the FP64 coarse and the literal table scan)
    for fc, fs in ((0, 0), (1, 1)):
        with v3db.option(v3db.OPT_FX_COARSE, fc), v3db.option(v3db.OPT_FX_SCAN, fs):
            sf = v3db.build_snapshot_fx(torch.from_numpy(fdb).cuda(), cfg.nlist, cfg.L, cfg.M, cfg.Ks,
                                        f.centroid_rows, f.codeword_rows)
            outf = v3db.query_batch_fx(sf, torch.from_numpy(fq).cuda(), cfg.nprobe, cfg.k)
            torch.cuda.synchronize()
            for key, exp in reff.items():
                assert np.array_equal(outf[key].cpu().numpy(), exp), (name, "fx16", fc, fs, key)
            sf.free()
    print("ok", name, flush=True)
print("lib", v3db._lib.LIB_PATH)
