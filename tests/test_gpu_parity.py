"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, element by element.

All arithmetic is integer, so the bar is bit-exact equality of every output: the snapshot
arrays (centroids, codebooks, ids, codes, counts, list_of), out_ids, out_dist,
trace_lists, trace_list_dist and trace_cand_dist.  Every scan kernel (the generic
query-major LUT scan, the rotated conflict-free LUT scan and the list-major tensor-core scan) is
checked.
"""
import numpy as np
import pytest

import oracle
from synth import generate, get_config

from .gpu_util import first_mismatch, oracle_queries

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FIELDS = ("centroids", "codebooks", "ids", "codes", "counts", "list_of")
ALGOS = {"auto": 0, "gen": 1, "rot": 2, "lm": 3}


@pytest.fixture(scope="module")
def v3db():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_03065_b200 import build as libbuild
    libbuild.build()
    from paper_2603_03065_b200 import v3db as mod
    return mod


def gpu_build(v3db, db, nlist, L, M, Ks, cent, code):
    return v3db.build_snapshot(torch.from_numpy(np.ascontiguousarray(db)).cuda(), nlist, L, M, Ks, cent, code)


def export_all(v3db, s):
    f = {"centroids": v3db.FIELD_CENTROIDS, "codebooks": v3db.FIELD_CODEBOOKS, "ids": v3db.FIELD_IDS,
         "codes": v3db.FIELD_CODES, "counts": v3db.FIELD_COUNTS, "list_of": v3db.FIELD_LIST_OF}
    return {k: v3db.snapshot_export(s, v) for k, v in f.items()}


def assert_snapshot_equal(v3db, s, ref):
    got = export_all(v3db, s)
    for name in FIELDS:
        exp = getattr(ref, name)
        assert np.array_equal(got[name], exp), f"snapshot {name}: {first_mismatch(got[name], exp)}"


def assert_query_equal(out, ref, rows=None, keys=None):
    for key, exp in ref.items():
        if keys is not None and key not in keys:
            continue
        got = out[key].cpu().numpy()
        if rows is not None:
            got = got[rows]
        assert np.array_equal(got, exp), f"{key}: {first_mismatch(got, exp)}"


_CACHE = {}


def config_case(name):
    """(cfg, inputs, oracle snapshot, oracle outputs for all queries) -- cached per module."""
    if name not in _CACHE:
        cfg = get_config(name)
        inp = generate(cfg)
        ref_s = oracle.build_snapshot(inp.db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows,
                                      inp.codeword_rows)
        ref = oracle_queries(ref_s, inp.queries, cfg.nprobe, cfg.k)
        _CACHE[name] = (cfg, inp, ref_s, ref)
    return _CACHE[name]


@pytest.mark.parametrize("algo", ["gen", "rot", "lm"])
@pytest.mark.parametrize("name", ["c0", "c1", "e2_basic", "e2_lowacc", "e2_large", "c4_mini"])
def test_full_parity_small_configs(v3db, name, algo):
    """Full snapshot + full query batch, bit-exact (C0, C1 and the paper's E2 shapes)."""
    cfg, inp, ref_s, ref = config_case(name)
    s = gpu_build(v3db, inp.db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    assert_snapshot_equal(v3db, s, ref_s)
    q = torch.from_numpy(inp.queries).cuda()
    out = v3db.query_batch(s, q, cfg.nprobe, cfg.k, trace=True, algo=ALGOS[algo])
    torch.cuda.synchronize()
    assert_query_equal(out, ref)
    s.free()


def run_case(v3db, db, queries, nlist, L, M, Ks, nprobe, k, cent, code, algos=("gen", "auto"), trace=True):
    ref_s = oracle.build_snapshot(db, nlist, L, M, Ks, cent, code)
    ref = oracle.query_batch(ref_s, queries, nprobe, k)
    s = gpu_build(v3db, db, nlist, L, M, Ks, cent, code)
    assert_snapshot_equal(v3db, s, ref_s)
    q = torch.from_numpy(np.ascontiguousarray(queries)).cuda()
    for algo in algos:
        out = v3db.query_batch(s, q, nprobe, k, trace=trace, algo=ALGOS[algo])
        torch.cuda.synchronize()
        assert_query_equal(out, ref, keys=None if trace else ("out_ids", "out_dist"))
    s.free()
    return ref_s, ref


def test_edge_k_equals_nsel_and_nprobe_equals_nlist(v3db):
    """k = N_sel (full sort) with n_probe = n_list."""
    rng = np.random.default_rng(11)
    N, D, nlist, L = 200, 16, 4, 64
    db = rng.integers(-60, 60, size=(N, D)).astype(np.int8)
    qs = rng.integers(-60, 60, size=(37, D)).astype(np.int8)
    run_case(v3db, db, qs, nlist, L, 4, 16, nlist, nlist * L, rng.choice(N, nlist, replace=False),
             np.stack([rng.choice(N, 16, replace=False) for _ in range(4)]))


def test_edge_fewer_than_k_valid(v3db):
    """Probed lists hold fewer than k valid candidates -> (-1, d_max) tail (R11)."""
    rng = np.random.default_rng(12)
    N, D, nlist, L = 40, 8, 8, 64
    db = rng.integers(-100, 100, size=(N, D)).astype(np.int8)
    qs = rng.integers(-100, 100, size=(19, D)).astype(np.int8)
    ref_s, ref = run_case(v3db, db, qs, nlist, L, 2, 8, 2, 100, rng.choice(N, nlist, replace=False),
                          np.stack([rng.choice(N, 8, replace=False) for _ in range(2)]))
    assert (ref["out_ids"] == -1).any()


def test_edge_all_identical_vectors(v3db):
    """Every vector identical: all distances tie, only the id tie-break orders (R10); lists
    with duplicate centroids lose every tie to the lowest index and stay empty (R2)."""
    N, D, nlist, L = 300, 8, 4, 100
    db = np.full((N, D), 7, np.int8)
    qs = np.vstack([np.full((1, D), 7, np.int8), np.full((1, D), -9, np.int8), np.arange(D, dtype=np.int8)[None]])
    run_case(v3db, db, qs, nlist, L, 4, 4, 3, 50, np.arange(nlist), np.stack([np.arange(4)] * 4))


def test_edge_outlier_list(v3db):
    """A query whose nearest list holds a single vector: the rotated scan's threshold stays
    open (fewer than k candidates seen) until later lists fill the buffer; still exact."""
    rng = np.random.default_rng(13)
    N, D, nlist, L = 3000, 8, 3, 2000
    db = rng.integers(-20, 20, size=(N, D)).astype(np.int8)
    db[0] = 120                                    # an outlier: its list holds (almost) only itself
    qs = np.vstack([np.full((4, D), 118, np.int8), rng.integers(-20, 20, size=(5, D)).astype(np.int8)])
    run_case(v3db, db, qs, nlist, L, 4, 32, 3, 10, [0, 1, 2], np.stack([rng.choice(N, 32, replace=False)] * 4))


@pytest.mark.parametrize("nq", [1, 67, 130])
def test_ragged_batch_sizes(v3db, nq):
    cfg, inp, ref_s, ref = config_case("c0")
    s = gpu_build(v3db, inp.db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    qs = np.vstack([inp.queries] * 3)[:nq]
    want = oracle.query_batch(ref_s, qs, cfg.nprobe, cfg.k)
    q = torch.from_numpy(np.ascontiguousarray(qs)).cuda()
    for algo in (1, 2, 3):
        out = v3db.query_batch(s, q, cfg.nprobe, cfg.k, algo=algo)
        torch.cuda.synchronize()
        assert_query_equal(out, want)
    s.free()


@pytest.mark.parametrize("name", ["c1", "c4_mini", "e2_basic"])
def test_rotated_w32_geometry(v3db, name, monkeypatch):
    """The wrap geometry (kLutW32) on shapes where AUTO picks the 64-column one: same bits."""
    cfg, inp, ref_s, ref = config_case(name)
    with v3db.option(v3db.OPT_LUT_W32, 1):
        s = gpu_build(v3db, inp.db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    out = v3db.query_batch(s, torch.from_numpy(inp.queries).cuda(), cfg.nprobe, cfg.k, algo=ALGOS["rot"])
    torch.cuda.synchronize()
    assert_query_equal(out, ref)
    s.free()


@pytest.mark.parametrize("M,d,k,geo", [(12, 4, 10, "w32"), (24, 4, 10, "w32"), (48, 2 * 4, 100, None),
                                       (96, 8, 100, None), (128, 4, 37, None), (12, 4, 10, None),
                                       (20, 4, 10, None), (24, 4, 10, None), (28, 4, 19, None)])
def test_rotated_group_decompositions(v3db, M, d, k, geo, monkeypatch):
    """W32 rotation groups of every size mix: 12 = 8+4, 24 = 16+8 (forced), 48 = 32+16, 96 = 3x32
    (512 consumer threads), 128 = 4x32; the P64 geometry with M not dividing 64 (12, 20, 24, 28:
    columns l + s hold subspace (l + s) mod M); ragged list fill and a ragged last chunk."""
    rng = np.random.default_rng(100 + M)
    N, D, nlist, L, Ks = 3000, M * d, 12, 300, 256
    db = rng.integers(-100, 100, size=(N, D)).astype(np.int8)
    qs = rng.integers(-100, 100, size=(41, D)).astype(np.int8)
    with v3db.option(v3db.OPT_LUT_W32, 1 if geo == "w32" else 0):
        run_case(v3db, db, qs, nlist, L, M, Ks, 5, k, rng.choice(N, nlist, replace=False),
                 np.stack([rng.choice(N, Ks, replace=False) for _ in range(M)]))


@pytest.mark.parametrize("k", [1, 7, 100, 333, 1024])
def test_rotated_topk_sizes(v3db, k):
    """Buffered top-k of the rotated scan for k from 1 to V3DB_MAX_K (compactions at every
    buffer size); C4's list shape (L = 768, M = 32)."""
    cfg, inp, ref_s, _ = config_case("c4_mini")
    qs = inp.queries[:48]
    want = oracle.query_batch(ref_s, qs, cfg.nprobe, k)
    s = gpu_build(v3db, inp.db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    out = v3db.query_batch(s, torch.from_numpy(qs).cuda(), cfg.nprobe, k, algo=ALGOS["rot"])
    torch.cuda.synchronize()
    assert_query_equal(out, want)
    s.free()


def test_empty_batch_and_trace_off_and_host_api(v3db):
    cfg, inp, ref_s, ref = config_case("c1")
    s = gpu_build(v3db, inp.db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    q = torch.from_numpy(inp.queries).cuda()
    # nq = 0 is a no-op
    v3db.query_batch(s, q[:0], cfg.nprobe, cfg.k)
    # trace off: same top-k
    for algo in (1, 2, 3):
        out = v3db.query_batch(s, q, cfg.nprobe, cfg.k, trace=False, algo=algo)
        torch.cuda.synchronize()
        assert_query_equal(out, ref, keys=("out_ids", "out_dist"))
    # host-buffer entry point (end-to-end path of bench.py)
    qh = torch.from_numpy(inp.queries).pin_memory()
    oh = v3db.alloc_outputs(s, cfg.Q, cfg.nprobe, cfg.k, trace=True, device="cpu", pin=True)
    v3db.query_batch_host(s, qh, cfg.nprobe, cfg.k, oh)   # Q = 10 000: pipelined in 4 sub-batches
    for key, exp in ref.items():
        assert np.array_equal(oh[key].numpy(), exp), key
    n = 9001                                                 # ragged sub-batches
    oh = v3db.alloc_outputs(s, n, cfg.nprobe, cfg.k, trace=True, device="cpu", pin=True)
    v3db.query_batch_host(s, qh[:n].contiguous(), cfg.nprobe, cfg.k, oh)
    for key, exp in ref.items():
        assert np.array_equal(oh[key].numpy(), exp[:n]), key
    oh = v3db.alloc_outputs(s, cfg.Q, cfg.nprobe, cfg.k, trace=False, device="cpu", pin=True)
    v3db.query_batch_host(s, qh, cfg.nprobe, cfg.k, oh)   # no trace: one batch
    assert_query_equal(oh, ref, keys=("out_ids", "out_dist"))
    s.free()


def test_determinism_across_runs_and_streams(v3db):
    cfg, inp, ref_s, ref = config_case("e2_large")
    s = gpu_build(v3db, inp.db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    q = torch.from_numpy(inp.queries).cuda()
    streams = [torch.cuda.Stream() for _ in range(2)]
    outs = []
    for st in streams:
        with torch.cuda.stream(st):
            outs.append(v3db.query_batch(s, q, cfg.nprobe, cfg.k, stream=st))
    torch.cuda.synchronize()
    for o in outs:
        assert_query_equal(o, ref)
    s.free()


def test_errors(v3db):
    cfg, inp, _, _ = config_case("c0")
    db = torch.from_numpy(inp.db).cuda()
    with pytest.raises(v3db.V3DBError, match="EINFEASIBLE"):
        v3db.build_snapshot(db, cfg.nlist, 100, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    bad = inp.centroid_rows.copy()
    bad[1] = bad[0]
    with pytest.raises(v3db.V3DBError, match="EINVAL"):
        v3db.build_snapshot(db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, bad, inp.codeword_rows)
    s = v3db.build_snapshot(db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    q = torch.from_numpy(inp.queries).cuda()
    with pytest.raises(v3db.V3DBError, match="EINVAL"):
        v3db.query_batch(s, q, cfg.nlist + 1, cfg.k)
    with pytest.raises(v3db.V3DBError, match="EINVAL"):
        v3db.query_batch(s, q, 1, cfg.L + 1)
    with pytest.raises(v3db.V3DBError, match="EINVAL"):
        v3db.query_batch(s, q, cfg.nprobe, cfg.k, algo=7)
    s.free()


def test_rotated_rejected_for_unsupported_shape(v3db):
    rng = np.random.default_rng(15)
    N, D = 300, 18
    db = rng.integers(-90, 90, size=(N, D)).astype(np.int8)
    s = gpu_build(v3db, db, 3, 200, 3, 8, [0, 1, 2], np.stack([np.arange(8)] * 3))
    with pytest.raises(v3db.V3DBError, match="EINVAL"):
        v3db.query_batch(s, torch.from_numpy(db[:5].copy()).cuda(), 2, 5, algo=ALGOS["rot"])
    s.free()


@pytest.mark.parametrize("name", ["c1", "e2_large"])
def test_coarse_mma_fallback_path(v3db, name, monkeypatch):
    """The mma.sync coarse kernel (used when the TMA/tcgen05 path does not apply) gives the
    same bit-exact snapshot and query results."""
    cfg, inp, ref_s, ref = config_case(name)
    with v3db.option(v3db.OPT_COARSE_SIMT, 1):
        s = gpu_build(v3db, inp.db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
        assert_snapshot_equal(v3db, s, ref_s)
        out = v3db.query_batch(s, torch.from_numpy(inp.queries).cuda(), cfg.nprobe, cfg.k)
        torch.cuda.synchronize()
    assert_query_equal(out, ref)
    s.free()


def test_odd_dim_generic_paths(v3db):
    """dim % 16 != 0 and d not in {4, 8, 16}: generic (non-TMA, byte-wise decode) paths."""
    rng = np.random.default_rng(14)
    N, D, nlist, L, M, Ks = 900, 18, 6, 200, 3, 32
    db = rng.integers(-90, 90, size=(N, D)).astype(np.int8)
    qs = rng.integers(-90, 90, size=(77, D)).astype(np.int8)
    run_case(v3db, db, qs, nlist, L, M, Ks, 3, 20, rng.choice(N, nlist, replace=False),
             np.stack([rng.choice(N, Ks, replace=False) for _ in range(M)]))


@pytest.mark.parametrize("name,nq", [("c0", 64), ("e2_lowacc", 16), ("e2_basic", 12), ("c4_mini", 6)])
def test_witness_batch(v3db, name, nq):
    """NEXT-2: the prover witness (§4.7) -- S^sorted_idx,dist, the selected literal LUT
    entries and S^sorted_item,dist -- bit-exact against oracle.witness, and consistent with the
    query path's trace and top-k."""
    cfg, inp, ref_s, ref = config_case(name)
    s = gpu_build(v3db, inp.db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    q = torch.from_numpy(np.ascontiguousarray(inp.queries[:nq])).cuda()
    w = v3db.witness_batch(s, q, cfg.nprobe)
    out = v3db.query_batch(s, q, cfg.nprobe, cfg.k)
    torch.cuda.synchronize()
    got = {k2: v.cpu().numpy() for k2, v in w.items()}
    for a in range(nq):
        order, od, ell, items, dists = oracle.witness(inp.queries[a], ref_s, cfg.nprobe)
        assert np.array_equal(got["list_order"][a], order), (a, first_mismatch(got["list_order"][a], order))
        assert np.array_equal(got["list_dist"][a], od), a
        assert np.array_equal(got["lut_sel"][a], ell), (a, first_mismatch(got["lut_sel"][a], ell))
        assert np.array_equal(got["cand_items"][a], items), (a, first_mismatch(got["cand_items"][a], items))
        assert np.array_equal(got["cand_dist"][a], dists), a
    assert np.array_equal(got["list_order"][:, :cfg.nprobe], out["trace_lists"].cpu().numpy())
    assert np.array_equal(got["cand_items"][:, :cfg.k], out["out_ids"].cpu().numpy())
    s.free()


@pytest.mark.parametrize("db,rows,L,expect", [
    ([3, 2, 1, 0, 10, 11, 20], [3, 4, 6], 3, [1, 0, 0, 0, 1, 1, 2]),
    ([0, 1, 2, 3, 4, 10, 11, 30], [0, 5, 7], 3, [0, 0, 0, 2, 1, 1, 1, 2]),
])
def test_rebalance_hand_examples_gpu(v3db, db, rows, L, expect):
    """NEXT-3: the paper's Alg. 1 on the hand-derived cases of tests/golden/rebalance_example.md."""
    x = np.array(db, np.int8)[:, None]
    stats = {}
    s = v3db.build_snapshot(torch.from_numpy(x).cuda(), len(rows), L, 1, 2, rows, [[0, 1]], rule=v3db.SHAPE_REBALANCE,
                            stats=stats)
    assert v3db.snapshot_export(s, v3db.FIELD_LIST_OF).tolist() == expect
    init = np.argmin((x.astype(np.int64) - x[rows].astype(np.int64).T) ** 2, axis=1)
    assert stats["moved"] == int((np.array(expect) != init).sum())
    s.free()


@pytest.mark.parametrize("name", ["c0_tight", "c1", "e2_basic", "e2_large"])
def test_rebalance_parity(v3db, name):
    """NEXT-3: snapshot shaped by Alg. 1 on the GPU == oracle, bit for bit, and
    the query path on it."""
    cfg = get_config("c0").with_(L=520) if name == "c0_tight" else get_config(name)
    inp = generate(cfg)
    ref_s = oracle.build_snapshot(inp.db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows,
                                  rule="rebalance")
    stats = {}
    s = v3db.build_snapshot(torch.from_numpy(inp.db).cuda(), cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows,
                            inp.codeword_rows, rule=v3db.SHAPE_REBALANCE, stats=stats)
    assert_snapshot_equal(v3db, s, ref_s)
    init = oracle.v3db_oracle.nearest_lists(inp.db, ref_s.centroids)
    assert stats["moved"] == int((ref_s.list_of != init).sum())
    qs = inp.queries[:128]
    want = oracle.query_batch(ref_s, qs, cfg.nprobe, cfg.k)
    out = v3db.query_batch(s, torch.from_numpy(np.ascontiguousarray(qs)).cuda(), cfg.nprobe, cfg.k)
    torch.cuda.synchronize()
    assert_query_equal(out, want)
    s.free()


# ---------------------------------------------------------------- list-major tensor-core scan

def test_lm_edge_all_identical_vectors(v3db):
    """Every D ties: tau (k-th smallest group minimum) equals every group's minimum, so every group
    is selected; the k winners come from the item-id radix pass among the ties (R10)."""
    N, D, nlist, L = 600, 32, 4, 200
    db = np.full((N, D), 7, np.int8)
    qs = np.vstack([np.full((1, D), 7, np.int8), np.full((1, D), -9, np.int8), np.arange(D, dtype=np.int8)[None]])
    run_case(v3db, db, qs, nlist, L, 4, 4, 3, 50, np.arange(nlist), np.stack([np.arange(4)] * 4),
             algos=("lm", "gen"))


def test_lm_edge_fewer_than_k_valid(v3db):
    """Fewer valid candidates than k (fewer valid groups than k): everything valid is returned,
    then (-1, d_max) (R11); lists shorter than one 32-slot group, tiles of padding only."""
    rng = np.random.default_rng(12)
    N, D, nlist, L = 40, 16, 8, 300
    db = rng.integers(-100, 100, size=(N, D)).astype(np.int8)
    qs = rng.integers(-100, 100, size=(19, D)).astype(np.int8)
    ref_s, ref = run_case(v3db, db, qs, nlist, L, 2, 8, 2, 100, rng.choice(N, nlist, replace=False),
                          np.stack([rng.choice(N, 8, replace=False) for _ in range(2)]), algos=("lm",))
    assert (ref["out_ids"] == -1).any()


def test_lm_edge_outlier_list(v3db):
    """A query whose nearest list holds a single vector (one valid group of one slot)."""
    rng = np.random.default_rng(13)
    N, D, nlist, L = 3000, 16, 3, 2000
    db = rng.integers(-20, 20, size=(N, D)).astype(np.int8)
    db[0] = 120
    qs = np.vstack([np.full((4, D), 118, np.int8), rng.integers(-20, 20, size=(5, D)).astype(np.int8)])
    run_case(v3db, db, qs, nlist, L, 4, 32, 3, 10, [0, 1, 2], np.stack([rng.choice(N, 32, replace=False)] * 4),
             algos=("lm",))


@pytest.mark.parametrize("D,M,L,nq", [(16, 4, 130, 300), (48, 12, 257, 70), (96, 24, 384, 41), (256, 32, 100, 33),
                                      (768, 96, 320, 20), (2048, 128, 64, 9)])
def test_lm_shapes(v3db, D, M, L, nq):
    """Dims below one 32-byte K step, ragged K panels (48, 96), several panels (256, 768, 2048 =
    the largest dim: 16 panels, NT = 32 pairs per item), L not a multiple of 128 (partial tiles,
    tiles of padding only), many queries per list (items split at NT)."""
    rng = np.random.default_rng(D + L)
    nlist = 12
    N = min(900, nlist * L * 9 // 10)
    db = rng.integers(-90, 90, size=(N, D)).astype(np.int8)
    qs = rng.integers(-90, 90, size=(nq, D)).astype(np.int8)
    run_case(v3db, db, qs, nlist, L, M, 16, 4, 37, rng.choice(N, nlist, replace=False),
             np.stack([rng.choice(N, 16, replace=False) for _ in range(M)]), algos=("lm",))


@pytest.mark.parametrize("nt", [32, 64, 128, 256])
def test_lm_items_per_pair_count(v3db, nt):
    """Every NT (pairs per work item: items split lists probed by more queries), same bits."""
    cfg, inp, ref_s, ref = config_case("c1")
    s = gpu_build(v3db, inp.db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    with v3db.option(v3db.OPT_LM_NT, nt):
        out = v3db.query_batch(s, torch.from_numpy(inp.queries).cuda(), cfg.nprobe, cfg.k, algo=ALGOS["lm"])
        torch.cuda.synchronize()
    assert_query_equal(out, ref)
    s.free()


@pytest.mark.parametrize("static", [0, 1])
@pytest.mark.parametrize("name", ["c1", "c4_mini", "e2_large"])
def test_lm_item_schedule(v3db, name, static):
    """The main kernel's CTAs draw their work items from a grid-wide counter (default) or take them
    round-robin (V3DB_OPT_LM_STATIC): whichever CTA runs an item, the bits are the same -- twice in a
    row, since the order the counter hands the items out differs from run to run."""
    cfg, inp, ref_s, ref = config_case(name)
    s = gpu_build(v3db, inp.db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    with v3db.option(v3db.OPT_LM_STATIC, static):
        for _ in range(2):
            out = v3db.query_batch(s, torch.from_numpy(inp.queries).cuda(), cfg.nprobe, cfg.k, algo=ALGOS["lm"])
            torch.cuda.synchronize()
            assert_query_equal(out, ref)
    s.free()


@pytest.mark.parametrize("static", [0, 1])
def test_lm_runs_of_empty_lists(v3db, static):
    """Hundreds of probed lists without a single vector (their centroid rows hold copies of one
    vector: the lowest list takes them all), between a few full ones: work items with no tile to
    load or multiply -- the TMA thread runs ahead through the item ring, bounded only by the ring --
    next to items of several tiles; every query probes every list."""
    rng = np.random.default_rng(77)
    N, D, nlist, L, M = 2400, 32, 300, 260, 8
    db = rng.integers(-90, 90, size=(N, D)).astype(np.int8)
    cent = rng.choice(N, nlist, replace=False)
    dup = np.ones(nlist, bool)
    dup[rng.choice(nlist, 12, replace=False)] = False      # 12 ordinary lists, 288 copies of one vector
    db[cent[dup]] = db[cent[dup][0]]
    qs = rng.integers(-90, 90, size=(150, D)).astype(np.int8)
    code = np.stack([rng.choice(N, 16, replace=False) for _ in range(M)])
    with v3db.option(v3db.OPT_LM_STATIC, static):
        ref_s, _ = run_case(v3db, db, qs, nlist, L, M, 16, nlist, 50, cent, code, algos=("lm",))
    assert (ref_s.counts == 0).sum() >= 200


@pytest.mark.parametrize("k", [1, 7, 100, 333, 1024])
def test_lm_topk_sizes(v3db, k):
    """The list-major Step-5 selection for k from 1 to V3DB_MAX_K (C4's list shape)."""
    cfg, inp, ref_s, _ = config_case("c4_mini")
    qs = inp.queries[:48]
    want = oracle.query_batch(ref_s, qs, cfg.nprobe, k)
    s = gpu_build(v3db, inp.db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    for trace in (True, False):
        out = v3db.query_batch(s, torch.from_numpy(qs).cuda(), cfg.nprobe, k, trace=trace, algo=ALGOS["lm"])
        torch.cuda.synchronize()
        assert_query_equal(out, want, keys=None if trace else ("out_ids", "out_dist"))
    s.free()


@pytest.mark.parametrize("mode", [0, 1, 4, 8, 32])
@pytest.mark.parametrize("name", ["c1", "c4_mini", "e2_large"])
def test_coarse_step2_paths(v3db, name, mode):
    """Steps 1-2: the single contraction pass keeping every 32-list block's two smallest keys
    (0, the default), the group-minimum pass followed by a second contraction pass (1) or by the
    recomputation of the selected groups with every group size (4, 8, 32) give the same bits."""
    cfg, inp, ref_s, ref = config_case(name)
    s = gpu_build(v3db, inp.db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    with v3db.option(v3db.OPT_COARSE_2PASS, mode):
        out = v3db.query_batch(s, torch.from_numpy(inp.queries).cuda(), cfg.nprobe, cfg.k)
        torch.cuda.synchronize()
    assert_query_equal(out, ref)
    s.free()


@pytest.mark.parametrize("mode", [0, 1])
def test_coarse_block_top2_adversarial(v3db, mode):
    """Single-pass Steps 1-2 where keeping two keys per block of 32 consecutive lists is not enough:
    (a) every block's 32 centroids are drawn around one centre, so a query's n_probe nearest lists
    share one block, which must be recomputed exactly; two centroids are duplicated (ties on d_i
    broken by the list index, R9); (b) every centroid is identical, so every block ties and the
    row overflows to the brute-force ranking.  Both equal the oracle (the second contraction pass,
    mode 1, beside it)."""
    rng = np.random.default_rng(21)
    D, nlist, L, nprobe, k = 32, 512, 64, 24, 10
    centres = rng.integers(-100, 100, size=(16, D))
    N = nlist * 8
    db = np.clip(centres[np.arange(N) // (N // 16)] + rng.integers(-3, 4, size=(N, D)), -127, 127).astype(np.int8)
    db[8 * 6] = db[8 * 5]                     # lists 5 and 6: one centroid twice
    cent = np.arange(0, N, 8)[:nlist]         # centroid i = row 8 i: block i // 32 <-> centre i // 32
    qs = np.clip(centres[rng.integers(0, 16, 40)] + rng.integers(-4, 5, size=(40, D)), -127, 127).astype(np.int8)
    qs = np.vstack([qs, db[8 * 5][None]])
    code = np.stack([rng.choice(N, 16, replace=False) for _ in range(4)])
    with v3db.option(v3db.OPT_COARSE_2PASS, mode):
        run_case(v3db, db, qs, nlist, L, 4, 16, nprobe, k, cent, code, algos=("lm", "gen"))
        with v3db.option(v3db.OPT_COARSE_KEYS, 4):
            run_case(v3db, db, qs, nlist, L, 4, 16, nprobe, k, cent, code, algos=("lm",))
        N2, nlist2 = 4096, 2048                  # (b) 64 blocks, every one tied
        db2 = np.full((N2, 16), 3, np.int8)
        qs2 = np.vstack([np.full((1, 16), 3, np.int8), np.arange(16, dtype=np.int8)[None]])
        run_case(v3db, db2, qs2, nlist2, 8, 4, 4, 40, 10, np.arange(nlist2), np.stack([np.arange(4)] * 4),
                 algos=("lm", "gen"))


@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("name", ["c1", "c4_mini", "e2_large", "e2_lowacc"])
def test_lm_select_paths(v3db, name, mode):
    """Step 5 of the list-major scan: auto (0), one CTA per query (1) and one warp per query (2)
    give the same bits (and the streaming path takes whatever either flags)."""
    cfg, inp, ref_s, ref = config_case(name)
    s = gpu_build(v3db, inp.db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    with v3db.option(v3db.OPT_SELECT_CTA, mode):
        out = v3db.query_batch(s, torch.from_numpy(inp.queries).cuda(), cfg.nprobe, cfg.k, algo=ALGOS["lm"])
        torch.cuda.synchronize()
    assert_query_equal(out, ref)
    s.free()


def test_lm_select_ties_beyond_window(v3db):
    """150 candidates tied at one distance (fewer than the per-query candidate cache, more than the
    last window bin holds): the warp selection flags the query and the streaming path ranks the
    ties by item id (R10)."""
    N, D, nlist, L = 150, 32, 2, 100
    db = np.full((N, D), 5, np.int8)
    qs = np.vstack([np.full((1, D), 5, np.int8), np.full((1, D), -3, np.int8)])
    with v3db.option(v3db.OPT_SELECT_CTA, 2):
        run_case(v3db, db, qs, nlist, L, 4, 4, 2, 10, np.arange(nlist), np.stack([np.arange(4)] * 4),
                 algos=("lm", "gen"))


@pytest.mark.parametrize("nprobe", [2, 3, 8])
def test_coarse_complete_blocks_adversarial(v3db, nprobe):
    """nprobe <= 8: the single pass keeps the smallest 2 / 4 / 8 >= nprobe keys of every 32-list
    block and the merge recomputes nothing (a list of the true top nprobe missing from its block
    would have >= nprobe smaller keys in that block alone).  Adversarial: every block's centroids
    are drawn around one centre, so a query's nearest lists share one block, with a duplicated
    centroid (ties on d_i broken by the list index, R9).  Equals the oracle; the two-pass path and
    two kept keys (recomputing the blocks) beside it."""
    rng = np.random.default_rng(23)
    D, nlist, L, k = 32, 512, 64, 10
    centres = rng.integers(-100, 100, size=(16, D))
    N = nlist * 8
    db = np.clip(centres[np.arange(N) // (N // 16)] + rng.integers(-3, 4, size=(N, D)), -127, 127).astype(np.int8)
    db[8 * 6] = db[8 * 5]
    db[8 * 40] = db[8 * 37]
    cent = np.arange(0, N, 8)[:nlist]
    qs = np.clip(centres[rng.integers(0, 16, 40)] + rng.integers(-4, 5, size=(40, D)), -127, 127).astype(np.int8)
    qs = np.vstack([qs, db[8 * 5][None], db[8 * 37][None]])
    code = np.stack([rng.choice(N, 16, replace=False) for _ in range(4)])
    run_case(v3db, db, qs, nlist, L, 4, 16, nprobe, k, cent, code, algos=("lm", "gen"))
    with v3db.option(v3db.OPT_COARSE_KEYS, 2):
        run_case(v3db, db, qs, nlist, L, 4, 16, nprobe, k, cent, code, algos=("lm",))
    with v3db.option(v3db.OPT_COARSE_2PASS, 1):
        run_case(v3db, db, qs, nlist, L, 4, 16, nprobe, k, cent, code, algos=("lm",))


@pytest.mark.parametrize("keys", [2, 4, 8])
@pytest.mark.parametrize("name", ["c1", "c4_mini", "e2_large"])
def test_coarse_keys_per_block(v3db, name, keys):
    """Single-pass Steps 1-2 keeping 2, 4 or 8 keys per 32-list block (8 only where nprobe <= 8,
    e.g. C1; elsewhere the option falls back to the automatic choice): the same bits."""
    cfg, inp, ref_s, ref = config_case(name)
    s = gpu_build(v3db, inp.db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    with v3db.option(v3db.OPT_COARSE_KEYS, keys):
        out = v3db.query_batch(s, torch.from_numpy(inp.queries).cuda(), cfg.nprobe, cfg.k)
        torch.cuda.synchronize()
    assert_query_equal(out, ref)
    s.free()
