"""GPU parity of NEXT-1, the paper's 16-bit fixed-point representation (
DESIGN.md R18/R19): encode -> build -> query through the C ABI (v3db_encode_fixed_point,
v3db_build_snapshot_fx, v3db_query_batch_fx) vs the oracle's fixed-point variant.  Integer work
throughout (int32 coordinates, int64 distances): the bar is bit-exact equality of every output.
"""
import time

import numpy as np
import pytest

import oracle
from synth import generate_float, get_config

from .gpu_util import first_mismatch, oracle_check, oracle_queries

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FIELDS = ("centroids", "codebooks", "ids", "codes", "counts", "list_of")
KEYS = ("out_ids", "out_dist", "trace_lists", "trace_list_dist", "trace_cand_dist")


@pytest.fixture(scope="module")
def v3db():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_03065_b200 import build as libbuild
    libbuild.build()
    from paper_2603_03065_b200 import v3db as mod
    return mod


def export_all(v3db, s):
    f = {"centroids": v3db.FIELD_CENTROIDS, "codebooks": v3db.FIELD_CODEBOOKS, "ids": v3db.FIELD_IDS,
         "codes": v3db.FIELD_CODES, "counts": v3db.FIELD_COUNTS, "list_of": v3db.FIELD_LIST_OF}
    return {k: v3db.snapshot_export(s, v) for k, v in f.items()}


def check_snapshot(v3db, s, ref_s):
    assert s.kind == v3db.KIND_FX16
    got = export_all(v3db, s)
    for name in FIELDS:
        exp = getattr(ref_s, name)
        assert np.array_equal(got[name], exp), f"snapshot {name}: {first_mismatch(got[name], exp)}"


def check_query(out, ref, keys=KEYS):
    for key in keys:
        got = out[key].cpu().numpy()
        assert got.dtype == ref[key].dtype, (key, got.dtype, ref[key].dtype)
        assert np.array_equal(got, ref[key]), f"{key}: {first_mismatch(got, ref[key])}"


def run_int32_case(v3db, db, qs, nlist, L, M, Ks, nprobe, k, cent, code):
    ref_s = oracle.build_snapshot(db, nlist, L, M, Ks, cent, code)
    ref = oracle_queries(ref_s, qs, nprobe, k)
    s = v3db.build_snapshot_fx(torch.from_numpy(np.ascontiguousarray(db)).cuda(), nlist, L, M, Ks, cent, code)
    check_snapshot(v3db, s, ref_s)
    out = v3db.query_batch_fx(s, torch.from_numpy(np.ascontiguousarray(qs)).cuda(), nprobe, k)
    check_query(out, ref)
    return ref_s, ref


_CACHE = {}


def fx_case(name):
    """(cfg, float inputs, oracle-encoded db / queries, oracle snapshot, oracle outputs)."""
    if name not in _CACHE:
        cfg = get_config(name)
        f = generate_float(cfg)
        db = oracle.encode_fixed_point(f.db, f.v_max)
        qs = oracle.encode_fixed_point(f.queries, f.v_max)
        ref_s = oracle.build_snapshot(db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, f.centroid_rows, f.codeword_rows)
        ref = oracle_queries(ref_s, qs, cfg.nprobe, cfg.k)
        _CACHE[name] = (cfg, f, db, qs, ref_s, ref)
    return _CACHE[name]


@pytest.mark.parametrize("name", ["c0", "c1", "e2_basic", "e2_lowacc", "e2_large", "c4_mini"])
def test_fx_end_to_end_parity(v3db, name):
    """float32 vectors -> GPU encoding -> GPU build -> GPU query, bit-exact against the oracle's
    encoding, build and query (every snapshot array, top-k and the whole witness trace)."""
    cfg, f, db, qs, ref_s, ref = fx_case(name)
    gdb = v3db.encode_fixed_point(torch.from_numpy(f.db).cuda(), f.v_max)
    gqs = v3db.encode_fixed_point(torch.from_numpy(f.queries).cuda(), f.v_max)
    assert np.array_equal(gdb.cpu().numpy(), db), first_mismatch(gdb.cpu().numpy(), db)
    assert np.array_equal(gqs.cpu().numpy(), qs)
    s = v3db.build_snapshot_fx(gdb, cfg.nlist, cfg.L, cfg.M, cfg.Ks, f.centroid_rows, f.codeword_rows)
    check_snapshot(v3db, s, ref_s)
    assert np.abs(v3db.snapshot_export(s, v3db.FIELD_CODEBOOKS)).max() > 127  # genuinely beyond int8
    out = v3db.query_batch_fx(s, gqs, cfg.nprobe, cfg.k)
    check_query(out, ref)
    out2 = v3db.query_batch_fx(s, gqs, cfg.nprobe, cfg.k, trace=False)
    check_query(out2, ref, keys=("out_ids", "out_dist"))


def test_fx_encoding_rounding_cases(v3db):
    """Hand-worked encodings (the oracle pin's values) and exact halves, on the GPU."""
    x = np.array([4.0, -4.0, 1.0, -1.0, 0.0, 3.9999], np.float32)
    got = v3db.encode_fixed_point(torch.from_numpy(x).cuda(), 4.0).cpu().numpy()
    assert got.tolist() == oracle.encode_fixed_point(x, 4.0).tolist()
    assert got[:5].tolist() == [65535, -65535, 16384, -16384, 0]
    # exact halves (v_max = 65535 makes y = v): half away from zero, not to even
    h = np.array([0.5, -0.5, 1.5, 2.5, -2.5, 65534.5], np.float32)
    got = v3db.encode_fixed_point(torch.from_numpy(h).cuda(), 65535.0).cpu().numpy()
    assert got.tolist() == [1, -1, 2, 3, -3, 65535]
    # the float32 neighbours of the halves: just below 1/2 rounds to 0 (floor(y + 0.5) would give 1)
    b = np.nextafter(np.float32(0.5), np.float32(0))
    n = np.array([b, -b, np.nextafter(np.float32(0.5), np.float32(1)), np.nextafter(np.float32(2.5), np.float32(0)),
                  np.nextafter(np.float32(1.5), np.float32(2))], np.float32)
    got = v3db.encode_fixed_point(torch.from_numpy(n).cuda(), 65535.0).cpu().numpy()
    assert got.tolist() == [0, 0, 1, 2, 2] == oracle.encode_fixed_point(n, 65535.0).tolist()
    rng = np.random.default_rng(5)
    y = (rng.standard_normal(1 << 20) * 3).astype(np.float32)
    vm = float(np.abs(y).max())
    g = v3db.encode_fixed_point(torch.from_numpy(y).cuda(), vm).cpu().numpy()
    assert np.array_equal(g, oracle.encode_fixed_point(y, vm))


def test_fx_extreme_magnitudes(v3db):
    """Coordinates at +-65535 (the range bound): the largest distances the keys must carry."""
    rng = np.random.default_rng(21)
    N, D, nlist, L, M, Ks = 600, 32, 12, 80, 8, 16
    db = rng.choice(np.array([-65535, -65534, 0, 65534, 65535], np.int32), size=(N, D)).astype(np.int32)
    qs = rng.choice(np.array([-65535, 65535], np.int32), size=(33, D)).astype(np.int32)
    run_int32_case(v3db, db, qs, nlist, L, M, Ks, 5, 40, rng.choice(N, nlist, replace=False),
                   np.stack([rng.choice(N, Ks, replace=False) for _ in range(M)]))


def test_fx_ties_and_fewer_than_k(v3db):
    """All vectors identical (every distance ties: the id tie-break orders, R10) and k above the
    valid count (-1, 2^63 - 1 tail)."""
    N, D, nlist, L = 300, 8, 4, 100
    db = np.full((N, D), 40000, np.int32)
    qs = np.vstack([np.full((1, D), 40000, np.int32), np.full((1, D), -9, np.int32),
                    (np.arange(D, dtype=np.int32) * 1000)[None]])
    _, ref = run_int32_case(v3db, db, qs, nlist, L, 4, 4, 3, 50, np.arange(nlist), np.stack([np.arange(4)] * 4))
    rng = np.random.default_rng(22)
    db = rng.integers(-65535, 65536, size=(40, 8)).astype(np.int32)
    qs = rng.integers(-65535, 65536, size=(19, 8)).astype(np.int32)
    _, ref = run_int32_case(v3db, db, qs, 8, 64, 2, 8, 2, 100, rng.choice(40, 8, replace=False),
                            np.stack([rng.choice(40, 8, replace=False) for _ in range(2)]))
    assert (ref["out_ids"] == -1).any() and (ref["out_dist"] == oracle.D_MAX_FX).any()


def test_fx_global_table_and_greedy_overflow(v3db):
    """M * Ks = 32768 (a 256 KiB int64 table does not fit in shared memory: the per-query table lives
    in global scratch) and a tight capacity with nlist > 64, so some vectors find all 64 ranked
    lists full (exact fallback)."""
    rng = np.random.default_rng(23)
    N, D, nlist, L, M, Ks = 4000, 128, 80, 52, 128, 256
    centres = rng.integers(-30000, 30000, size=(3, D))
    db = (centres[rng.integers(0, 3, N)] + rng.integers(-3000, 3000, size=(N, D))).astype(np.int32)
    qs = (centres[rng.integers(0, 3, 25)] + rng.integers(-3000, 3000, size=(25, D))).astype(np.int32)
    run_int32_case(v3db, db, qs, nlist, L, M, Ks, 6, 30, rng.choice(N, nlist, replace=False),
                   np.stack([rng.choice(N, Ks, replace=False) for _ in range(M)]))


@pytest.mark.parametrize("nq", [0, 1, 67])
def test_fx_ragged_batches(v3db, nq):
    cfg, f, db, qs, ref_s, ref = fx_case("e2_basic")
    s = v3db.build_snapshot_fx(torch.from_numpy(db).cuda(), cfg.nlist, cfg.L, cfg.M, cfg.Ks, f.centroid_rows,
                               f.codeword_rows)
    out = v3db.query_batch_fx(s, torch.from_numpy(np.ascontiguousarray(qs[:nq])).cuda(), cfg.nprobe, cfg.k)
    for key in KEYS:
        assert np.array_equal(out[key].cpu().numpy(), ref[key][:nq]), key


def test_fx_errors(v3db):
    cfg, f, db, qs, ref_s, ref = fx_case("c0")
    gdb = torch.from_numpy(db).cuda()
    bad = gdb.clone()
    bad[3, 2] = 65536
    with pytest.raises(v3db.V3DBError, match="EINVAL"):
        v3db.build_snapshot_fx(bad, cfg.nlist, cfg.L, cfg.M, cfg.Ks, f.centroid_rows, f.codeword_rows)
    s = v3db.build_snapshot_fx(gdb, cfg.nlist, cfg.L, cfg.M, cfg.Ks, f.centroid_rows, f.codeword_rows)
    gq = torch.from_numpy(qs).cuda()
    badq = gq.clone()
    badq[0, 0] = -65536
    with pytest.raises(v3db.V3DBError, match="EINVAL"):
        v3db.query_batch_fx(s, badq, cfg.nprobe, cfg.k)
    with pytest.raises(v3db.V3DBError, match="EINVAL"):   # int8 entry point on a fixed-point snapshot
        v3db.query_batch(s, gq.to(torch.int8), cfg.nprobe, cfg.k)
    with pytest.raises(v3db.V3DBError, match="EINVAL"):
        v3db.witness_batch(s, gq.to(torch.int8), cfg.nprobe)
    with pytest.raises(v3db.V3DBError, match="EINVAL"):
        v3db.query_batch_fx(s, gq, cfg.nprobe, cfg.nprobe * cfg.L + 1)
    from synth import generate
    inp = generate(cfg)
    s8 = v3db.build_snapshot(torch.from_numpy(inp.db).cuda(), cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows,
                             inp.codeword_rows)
    assert s8.kind == v3db.KIND_INT8
    with pytest.raises(v3db.V3DBError, match="EINVAL"):   # fixed-point entry point on an int8 snapshot
        v3db.query_batch_fx(s8, gq, cfg.nprobe, cfg.k)
    with pytest.raises(v3db.V3DBError, match="EINVAL"):
        v3db.encode_fixed_point(torch.zeros(4, device="cuda"), 0.0)


def test_fx_heavy_ties_and_wide_nprobe(v3db):
    """Binary coordinates scaled to the fixed-point range: distances take few values, so ties at
    the k-th distance straddle the per-warp lists (the exact id re-selection path); nprobe = 150 >
    128 also takes the two-kernel Step-1/2 path (distance matrix + per-row top-R)."""
    rng = np.random.default_rng(24)
    N, D, nlist, L, M, Ks = 3000, 8, 200, 40, 4, 16
    db = (rng.integers(0, 2, size=(N, D)) * 65535).astype(np.int32)
    qs = (rng.integers(0, 2, size=(41, D)) * 65535).astype(np.int32)
    cent = rng.choice(N, nlist, replace=False)
    code = np.stack([rng.choice(N, Ks, replace=False) for _ in range(M)])
    run_int32_case(v3db, db, qs, nlist, L, M, Ks, 3, 25, cent, code)
    run_int32_case(v3db, db, qs, nlist, L, M, Ks, 150, 333, cent, code)


@pytest.mark.parametrize("M,d,Ks", [(24, 4, 256), (48, 2, 256), (16, 8, 256), (32, 4, 64), (96, 8, 256),
                                    (64, 2, 256), (8, 4, 256)])
def test_fx_scan_shapes(v3db, M, d, Ks):
    """Every scan instantiation: the rotated table (Ks = 256) with groups of 16 only (M = 16, 64, 96),
    16 + a trailing group of 8 (M = 24) and 8 only (M = 8); M = 48 (generic loop over the canonical
    codes although a rotated copy exists); Ks = 64 (runtime table stride, canonical codes)."""
    rng = np.random.default_rng(25 + M)
    D = M * d
    N, nlist, L = 3000, 24, 160
    centres = rng.integers(-40000, 40000, size=(6, D))
    db = np.clip(centres[rng.integers(0, 6, N)] + rng.integers(-9000, 9000, size=(N, D)), -65535, 65535).astype(np.int32)
    qs = np.clip(centres[rng.integers(0, 6, 70)] + rng.integers(-9000, 9000, size=(70, D)), -65535, 65535).astype(np.int32)
    run_int32_case(v3db, db, qs, nlist, L, M, Ks, 5, 37, rng.choice(N, nlist, replace=False),
                   np.stack([rng.choice(N, Ks, replace=False) for _ in range(M)]))


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_fx_full_size_parity(v3db, name):
    """BASELINE.json's full sizes in bench.py --precision fx16's launch configuration (whole batch,
    trace on) against the oracle's OWN fixed-point build: the GPU encoding equals the oracle's on
    every query and on sampled database rows, every exported snapshot array equals the oracle's
    build from the oracle's encoding, and the oracle's query on its snapshot reproduces every query
    row -- top-k, probed lists, their distances and the whole int64 candidate trace -- bit for bit
    (shards of 4096 rows)."""
    cfg = get_config(name)
    t0 = time.time()
    f = generate_float(cfg)
    rng = np.random.default_rng(2027)
    gdb = v3db.encode_fixed_point(torch.from_numpy(f.db).cuda(), f.v_max)
    rows = np.unique(np.concatenate([rng.choice(cfg.N, 4096, replace=False), [0, cfg.N - 1]]))
    db = oracle.encode_fixed_point(f.db, f.v_max)
    assert np.array_equal(gdb[torch.from_numpy(rows).cuda()].cpu().numpy(), db[rows])
    qs = oracle.encode_fixed_point(f.queries, f.v_max)
    gq = v3db.encode_fixed_point(torch.from_numpy(f.queries).cuda(), f.v_max)
    assert np.array_equal(gq.cpu().numpy(), qs)
    s = v3db.build_snapshot_fx(gdb, cfg.nlist, cfg.L, cfg.M, cfg.Ks, f.centroid_rows, f.codeword_rows)
    del gdb
    snap = export_all(v3db, s)
    t1 = time.time()
    ref_s = oracle.build_snapshot(db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, f.centroid_rows, f.codeword_rows)
    t2 = time.time()
    del db
    for key in ("centroids", "codebooks", "ids", "codes", "counts", "list_of"):
        got, exp = snap[key], getattr(ref_s, key)
        assert got.dtype == exp.dtype and np.array_equal(got, exp), f"{name} fx snapshot {key}: {first_mismatch(got, exp)}"
    del snap
    out = v3db.query_batch_fx(s, gq, cfg.nprobe, cfg.k, trace=True)
    torch.cuda.synchronize()
    s.free()
    t3 = time.time()
    for lo in range(0, cfg.Q, 4096):
        rr = np.arange(lo, min(cfg.Q, lo + 4096))
        got = {key: v[lo:lo + len(rr)].cpu().numpy() for key, v in out.items()}
        bad = oracle_check(ref_s, qs, cfg.nprobe, cfg.k, got, rows=rr)
        assert not bad, f"{name} fx: {bad[:3]}"
    print(f"[{name} fx16] generate + encode + GPU build {t1 - t0:.1f}s, oracle build {t2 - t1:.1f}s, GPU query "
          f"{t3 - t2:.1f}s, oracle queries + compare {time.time() - t3:.1f}s", flush=True)


def test_fx_host_entry(v3db):
    """v3db_query_batch_fx_host (HOST float32 queries, encoding inside the call) equals the oracle."""
    cfg, f, db, qs, ref_s, ref = fx_case("e2_large")
    s = v3db.build_snapshot_fx(torch.from_numpy(db).cuda(), cfg.nlist, cfg.L, cfg.M, cfg.Ks, f.centroid_rows,
                               f.codeword_rows)
    oh = v3db.alloc_outputs_fx(s, cfg.Q, cfg.nprobe, cfg.k, trace=True, device="cpu", pin=True)
    v3db.query_batch_fx_host(s, torch.from_numpy(f.queries), f.v_max, cfg.nprobe, cfg.k, oh)
    check_query(oh, ref)
    cfg1, f1, db1, qs1, ref_s1, ref1 = fx_case("c1")          # Q = 10 000: pipelined sub-batches
    s1 = v3db.build_snapshot_fx(torch.from_numpy(db1).cuda(), cfg1.nlist, cfg1.L, cfg1.M, cfg1.Ks, f1.centroid_rows,
                                f1.codeword_rows)
    oh1 = v3db.alloc_outputs_fx(s1, cfg1.Q, cfg1.nprobe, cfg1.k, trace=True, device="cpu", pin=True)
    v3db.query_batch_fx_host(s1, torch.from_numpy(f1.queries), f1.v_max, cfg1.nprobe, cfg1.k, oh1)
    check_query(oh1, ref1)
    oh2 = v3db.alloc_outputs_fx(s, cfg.Q, cfg.nprobe, cfg.k, trace=False, device="cpu")
    v3db.query_batch_fx_host(s, torch.from_numpy(f.queries), f.v_max, cfg.nprobe, cfg.k, oh2)
    check_query(oh2, ref, keys=("out_ids", "out_dist"))


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("name", ["c1", "e2_large", "c4_mini"])
def test_fx_coarse_paths(v3db, name, mode):
    """Fixed-point Steps 1-2 (query and the build's B2 ranking): the tensor-core kernel (0, three
    int8 limbs per coordinate, five int32 accumulators, exact int64 keys) and the FP64-FMA kernel (1)
    give the oracle's bits."""
    cfg, f, db, qs, ref_s, ref = fx_case(name)
    with v3db.option(v3db.OPT_FX_COARSE, mode):
        s = v3db.build_snapshot_fx(torch.from_numpy(db).cuda(), cfg.nlist, cfg.L, cfg.M, cfg.Ks, f.centroid_rows,
                                   f.codeword_rows)
        check_snapshot(v3db, s, ref_s)
        out = v3db.query_batch_fx(s, torch.from_numpy(qs).cuda(), cfg.nprobe, cfg.k)
        check_query(out, ref)


def test_fx_coarse_tc_adversarial(v3db):
    """Tensor-core fixed-point Steps 1-2 where two keys per block of 32 lists are not enough:
    (a) every block's centroids drawn around one centre at the +-65535 extremes (a query's nearest
    lists share one block: exact recomputation; a duplicated centroid: ties on d_i broken by the
    list index, R9); (b) every centroid identical: every block ties, the brute-force ranking."""
    rng = np.random.default_rng(25)
    D, nlist, L = 32, 512, 64
    centres = rng.choice(np.array([-65535, -40000, 0, 40000, 65535]), size=(16, D))
    N = nlist * 8
    db = np.clip(centres[np.arange(N) // (N // 16)] + rng.integers(-300, 301, size=(N, D)), -65535, 65535).astype(np.int32)
    db[8 * 6] = db[8 * 5]
    cent = np.arange(0, N, 8)[:nlist]
    qs = np.clip(centres[rng.integers(0, 16, 30)] + rng.integers(-400, 401, size=(30, D)), -65535, 65535).astype(np.int32)
    qs = np.vstack([qs, db[8 * 5][None]])
    code = np.stack([rng.choice(N, 16, replace=False) for _ in range(4)])
    run_int32_case(v3db, db, qs, nlist, L, 4, 16, 24, 10, cent, code)
    db2 = np.full((4096, 16), 30000, np.int32)
    qs2 = np.vstack([np.full((1, 16), 30000, np.int32), (np.arange(16, dtype=np.int32) * 4000)[None]])
    run_int32_case(v3db, db2, qs2, 2048, 8, 4, 4, 40, 10, np.arange(2048), np.stack([np.arange(4)] * 4))


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("name", ["c0", "c1", "e2_large", "c4_mini"])
def test_fx_scan_paths(v3db, name, mode):
    """Fixed-point Steps 3-5: the list-major tensor-core scan (0: three int8 limbs per coordinate,
    five int32 accumulators per tile, int64 D, the int64 instantiation of Step 5) and the literal
    per-query int64 LUT scan (1) give the oracle's bits, top-k and the whole trace."""
    cfg, f, db, qs, ref_s, ref = fx_case(name)
    s = v3db.build_snapshot_fx(torch.from_numpy(db).cuda(), cfg.nlist, cfg.L, cfg.M, cfg.Ks, f.centroid_rows,
                               f.codeword_rows)
    with v3db.option(v3db.OPT_FX_SCAN, mode):
        out = v3db.query_batch_fx(s, torch.from_numpy(qs).cuda(), cfg.nprobe, cfg.k)
        check_query(out, ref)
        out2 = v3db.query_batch_fx(s, torch.from_numpy(qs).cuda(), cfg.nprobe, cfg.k, trace=False)
        check_query(out2, ref, keys=("out_ids", "out_dist"))


@pytest.mark.parametrize("L", [130, 257, 384])
def test_fx_list_major_shapes(v3db, L):
    """List capacities that are not multiples of the 128-slot tile, odd (the P terms then come from
    global memory) and lists shorter than L (padding-only tiles), with extreme coordinates."""
    rng = np.random.default_rng(26)
    N, D, nlist, M, Ks = 600, 32, 6, 8, 16
    db = rng.choice(np.array([-65535, -30000, 0, 30000, 65535], np.int32), size=(N, D)).astype(np.int32)
    db[: N // 2] += rng.integers(-100, 100, size=(N // 2, D)).astype(np.int32)
    db = np.clip(db, -65535, 65535).astype(np.int32)
    qs = rng.integers(-65535, 65536, size=(45, D)).astype(np.int32)
    run_int32_case(v3db, db, qs, nlist, L, M, Ks, 4, 50, rng.choice(N, nlist, replace=False),
                   np.stack([rng.choice(N, Ks, replace=False) for _ in range(M)]))
