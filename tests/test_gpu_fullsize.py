"""GPU parity at BASELINE.json's full sizes (C1-C4), in the launch configuration bench.py times
(the whole query batch, V3DB_SCAN_AUTO, trace on), against the oracle's OWN build.

The oracle builds its snapshot from the same seeded inputs (B1-B6; C4: 10^7
vectors ranked against 16 384 lists on the host cores) and every exported snapshot array of the GPU
build must equal it.  The oracle's query (Steps 1-5) then runs on the oracle's
snapshot for EVERY query row of the batch, in shards of 2048 rows, and every output -- top-k ids
and distances, probed lists, their distances and the whole candidate trace (3.2 GB at C4) -- must
equal the GPU's bit for bit, for the list-major scan (AUTO) and the rotated-LUT scan.
"""
import time

import numpy as np
import pytest

import oracle
from synth import generate, get_config

from .gpu_util import first_mismatch, oracle_check

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FIELDS = ("centroids", "codebooks", "ids", "codes", "counts", "list_of")
SHARD = 4096


@pytest.fixture(scope="module")
def v3db():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_03065_b200 import build as libbuild
    libbuild.build()
    from paper_2603_03065_b200 import v3db as mod
    return mod


def export(v3db, s):
    f = {"centroids": v3db.FIELD_CENTROIDS, "codebooks": v3db.FIELD_CODEBOOKS, "ids": v3db.FIELD_IDS,
         "codes": v3db.FIELD_CODES, "counts": v3db.FIELD_COUNTS, "list_of": v3db.FIELD_LIST_OF}
    return {k: v3db.snapshot_export(s, v) for k, v in f.items()}


def compare_all_rows(name, outs, ref_s, queries, nprobe, k):
    """Every query row of every GPU output dict in `outs` vs the oracle on ref_s, in shards of
    SHARD rows (the workers compare in place: tests/gpu_util.oracle_check)."""
    Q = queries.shape[0]
    for lo in range(0, Q, SHARD):
        rows = np.arange(lo, min(Q, lo + SHARD))
        for label, out in outs.items():
            got = {key: v[lo:lo + len(rows)].cpu().numpy() for key, v in out.items()}
            bad = oracle_check(ref_s, queries, nprobe, k, got, rows=rows)
            assert not bad, f"{name} {label}: {bad[:3]}"


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_full_size_parity(v3db, name):
    cfg = get_config(name)
    t0 = time.time()
    inp = generate(cfg)
    s = v3db.build_snapshot(torch.from_numpy(inp.db).cuda(), cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows,
                            inp.codeword_rows)
    snap = export(v3db, s)
    t1 = time.time()
    ref_s = oracle.build_snapshot(inp.db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    t2 = time.time()
    for key in FIELDS:
        got, exp = snap[key], getattr(ref_s, key)
        assert got.dtype == exp.dtype and np.array_equal(got, exp), f"{name} snapshot {key}: {first_mismatch(got, exp)}"
    del snap
    # the bench's launch (the whole batch, AUTO = list-major scan, trace on), and the rotated-LUT scan
    q = torch.from_numpy(inp.queries).cuda()
    outs = {"auto": v3db.query_batch(s, q, cfg.nprobe, cfg.k, trace=True),
            "rot": v3db.query_batch(s, q, cfg.nprobe, cfg.k, trace=True, algo=v3db.SCAN_ROTATED)}
    rng = np.random.default_rng(2026)
    wq = [int(rng.integers(cfg.Q)) for _ in range(2)]          # two "challenged" queries (NEXT-2)
    w = v3db.witness_batch(s, q[wq].contiguous(), cfg.nprobe)
    torch.cuda.synchronize()
    s.free()
    t3 = time.time()
    compare_all_rows(name, outs, ref_s, inp.queries, cfg.nprobe, cfg.k)
    print(f"[{name}] generate + GPU build {t1 - t0:.1f}s, oracle build {t2 - t1:.1f}s, GPU queries {t3 - t2:.1f}s, "
          f"oracle queries + compare {time.time() - t3:.1f}s", flush=True)
    for a, qi in enumerate(wq):
        exp = oracle.witness(inp.queries[qi], ref_s, cfg.nprobe)
        for key, e in zip(("list_order", "list_dist", "lut_sel", "cand_items", "cand_dist"), exp):
            got = w[key][a].cpu().numpy()
            assert np.array_equal(got, e), f"{name} witness {key}: {first_mismatch(got, e)}"
