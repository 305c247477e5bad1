"""GPU parity at BASELINE.json's full sizes (C1-C4), in the launch configuration bench.py times
(the whole query batch, V3DB_SCAN_AUTO, trace on): every query row of the batch (the candidate
trace of every row for C1-C3, of 2048 sampled rows for C4), the oracle run on a process pool.

At these sizes the oracle's own build is too slow to run in a test (C4: 2.1e13 MACs to rank), so
the GPU-built snapshot is verified directly against the build rules instead (SURVEY.md §8(c)
B1-B6, pins P7/P8): exact structure, every centroid and codeword, the greedy placement replayed
for sampled vectors, the PQ codes of sampled slots by brute force.  The oracle's query (Steps
1-5) then runs on that verified snapshot for every query and every output --
top-k ids and distances, probed lists, their distances and the candidate trace -- must equal the
GPU's bit for bit.
"""
import numpy as np
import pytest

import oracle
from synth import generate, get_config

from .gpu_util import first_mismatch, oracle_queries_all
from .snapshot_checks import check_snapshot

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


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


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_full_size_sampled_parity(v3db, name):
    cfg = get_config(name)
    inp = generate(cfg)
    rng = np.random.default_rng(2026)
    s = v3db.build_snapshot(torch.from_numpy(inp.db).cuda(), cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows,
                            inp.codeword_rows)
    snap = export(v3db, s)
    check_snapshot(cfg, inp, snap, rng)
    # the bench's launch: the whole batch, AUTO scan, trace on
    q = torch.from_numpy(inp.queries).cuda()
    out = v3db.query_batch(s, q, cfg.nprobe, cfg.k, trace=True)
    wq = [int(rng.integers(cfg.Q)) for _ in range(2)]          # two "challenged" queries (NEXT-2)
    w = v3db.witness_batch(s, q[wq].contiguous(), cfg.nprobe)
    torch.cuda.synchronize()
    s.free()
    ref_snap = oracle.Snapshot(snap["centroids"], snap["codebooks"], snap["ids"], snap["codes"], snap["counts"],
                               snap["list_of"])
    # EVERY query row: top-k ids and distances, probed lists and their distances; the candidate
    # trace for every row up to 2^28 entries (C1-C3), else for 2048 sampled rows (C4: 3.2 GB)
    if cfg.Q * cfg.nprobe * cfg.L <= (1 << 28):
        trace_rows = np.arange(cfg.Q)
    else:
        trace_rows = np.unique(np.concatenate([rng.choice(cfg.Q, 2046, replace=False), [0, cfg.Q - 1]]))
    full, tr_rows, tr_vals = oracle_queries_all(ref_snap, inp.queries, cfg.nprobe, cfg.k, trace_rows)
    for key, exp in full.items():
        got = out[key].cpu().numpy()
        assert np.array_equal(got, exp), f"{name} {key}: {first_mismatch(got, exp)}"
    got = out["trace_cand_dist"][torch.from_numpy(tr_rows).cuda()].cpu().numpy()
    assert np.array_equal(got, tr_vals), f"{name} trace_cand_dist: {first_mismatch(got, tr_vals)}"
    for a, qi in enumerate(wq):
        exp = oracle.witness(inp.queries[qi], ref_snap, cfg.nprobe)
        for key, e in zip(("list_order", "list_dist", "lut_sel", "cand_items", "cand_dist"), exp):
            got = w[key][a].cpu().numpy()
            assert np.array_equal(got, e), f"{name} witness {key}: {first_mismatch(got, e)}"
