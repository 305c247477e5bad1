"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, element by element.

All arithmetic is integer, so the bar is bit-exact equality of every output: the snapshot
arrays (centroids, codebooks, ids, codes, counts, list_of), out_ids, out_dist,
trace_lists, trace_list_dist and trace_cand_dist.
"""
import numpy as np
import pytest

import oracle
from synth import generate, get_config

from .gpu_util import first_mismatch, oracle_queries

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FIELDS = ("centroids", "codebooks", "ids", "codes", "counts", "list_of")


@pytest.fixture(scope="module")
def v3db():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_03065_b200 import build as libbuild
    libbuild.build()
    from paper_2603_03065_b200 import v3db as mod
    return mod


def gpu_build(v3db, inp, cfg):
    db = torch.from_numpy(inp.db).cuda()
    return v3db.build_snapshot(db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)


def export_all(v3db, s):
    f = {"centroids": v3db.FIELD_CENTROIDS, "codebooks": v3db.FIELD_CODEBOOKS, "ids": v3db.FIELD_IDS,
         "codes": v3db.FIELD_CODES, "counts": v3db.FIELD_COUNTS, "list_of": v3db.FIELD_LIST_OF}
    return {k: v3db.snapshot_export(s, v) for k, v in f.items()}


def assert_snapshot_equal(v3db, s, ref):
    got = export_all(v3db, s)
    for name in FIELDS:
        exp = getattr(ref, name)
        assert np.array_equal(got[name], exp), f"snapshot {name}: {first_mismatch(got[name], exp)}"


def assert_query_equal(out, ref, rows=None):
    for key, exp in ref.items():
        got = out[key].cpu().numpy()
        if rows is not None:
            got = got[rows]
        assert np.array_equal(got, exp), f"{key}: {first_mismatch(got, exp)}"


@pytest.mark.parametrize("name", ["c0", "c1", "e2_basic", "e2_lowacc", "e2_large"])
def test_full_parity_small_configs(v3db, name):
    """Full snapshot + full query batch, bit-exact (C0, C1 and the paper's E2 shapes)."""
    cfg = get_config(name)
    inp = generate(cfg)
    ref_s = oracle.build_snapshot(inp.db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    s = gpu_build(v3db, inp, cfg)
    assert_snapshot_equal(v3db, s, ref_s)
    q = torch.from_numpy(inp.queries).cuda()
    out = v3db.query_batch(s, q, cfg.nprobe, cfg.k, trace=True)
    torch.cuda.synchronize()
    ref = oracle_queries(ref_s, inp.queries, cfg.nprobe, cfg.k)
    assert_query_equal(out, ref)
