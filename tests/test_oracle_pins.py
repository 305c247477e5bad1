"""Pins of the CPU oracle against things other than itself (no GPU needed).

Each test names the paper passage (or SPEC.md example derived from it) and what kind of
pin it is: a hand-derived worked example (tests/golden/), a closed form, an independent
library routine, a special case that reduces to exact k-NN, or brute force on tiny inputs.
"""
import json
import os

import numpy as np
import pytest
from scipy.spatial.distance import cdist

import oracle
from oracle import v3db_oracle as vo

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- SPEC.md worked examples

def test_spec_dist_examples():
    for ex in _load("spec_examples.json")["dist"]:
        assert oracle.dist(ex["x"], ex["y"]) == ex["expect"], ex["cite"]


def test_spec_step2_examples():
    for ex in _load("spec_examples.json")["step2"]:
        got = oracle.step2_probe_select(np.array(ex["d"], np.int64), ex["nprobe"])
        assert got.tolist() == ex["expect"], ex["cite"]


def test_spec_step4_examples():
    # M = 2, Ks = 5, one list with one slot whose codes select LUT entries 3 and 4.
    for ex in _load("spec_examples.json")["step4"]:
        lut = np.zeros((1, 2, 5), np.int64)
        lut[0, 0, 1] = ex["lut_entries"][0]
        lut[0, 1, 4] = ex["lut_entries"][1]
        s = vo.Snapshot(
            centroids=np.zeros((1, 2), np.int8), codebooks=np.zeros((2, 5, 1), np.int8),
            ids=np.array([[0 if ex["f"] else -1]], np.int32),
            codes=np.array([[[1, 4]]], np.uint8), counts=np.array([ex["f"]], np.int32),
            list_of=np.zeros(1, np.int32))
        got = oracle.step4_candidate_distances(s, np.array([0]), lut)
        assert got.tolist() == [[ex["expect"]]], ex["cite"]


def test_spec_step5_examples():
    for ex in _load("spec_examples.json")["step5"]:
        items, _ = oracle.step5_topk(np.array(ex["items"]), np.array(ex["dists"]), ex["k"])
        assert items.tolist() == ex["expect_items"], ex["cite"]


# ---------------------------------------------------------------- hand-derived end-to-end example

@pytest.mark.parametrize("case_idx", [0, 1])
def test_hand_example(case_idx):
    g = _load("hand_example.json")
    case = g["cases"][case_idx]
    s = oracle.build_snapshot(np.array(g["db"], np.int8), 2, case["L"], g["M"], g["Ks"],
                              g["centroid_rows"], g["codeword_rows"])
    exp = case["expect_snapshot"]
    assert s.centroids.tolist() == exp["centroids"]
    assert s.codebooks.tolist() == exp["codebooks"]
    assert s.ids.tolist() == exp["ids"]
    assert s.codes.tolist() == exp["codes"]
    assert s.counts.tolist() == exp["counts"]
    q = np.array(g["query"], np.int8)
    for qc in case["queries"]:
        ids, dd, probes, dP, cand = oracle.query(q, s, qc["nprobe"], qc["k"])
        if "step1_d" in qc:
            assert oracle.step1_centroid_distances(q, s).tolist() == qc["step1_d"]
        assert probes.tolist() == qc["probes"]
        if "lut" in qc:
            assert oracle.step3_adc_tables(q, s, probes).tolist() == qc["lut"]
        if "cand" in qc:
            assert cand.tolist() == qc["cand"]
        assert ids.tolist() == qc["out_ids"]
        assert dd.tolist() == qc["out_dist"]


def test_codeword_saturation_by_hand():
    """R5: a residual coordinate outside [-127,127] is saturated in the codebook but not
    in the encoded residual.  db row 1 = [127], centroid row 0 = [-100]: residual 227 ->
    codeword 127; encoding residual 227 against {0, 127} picks 127 (c = 1)."""
    db = np.array([[-100], [127], [-100 + 0]], np.int8)
    # rows 0 and 2 are identical; centroid row 0 only (nlist = 1, L = 3)
    s = oracle.build_snapshot(db, 1, 3, 1, 2, [0], [[0, 1]])
    assert s.codebooks.tolist() == [[[0], [127]]]
    assert s.codes[0, :, 0].tolist() == [0, 1, 0]
    # query q = [27]: LUT_{0,0,c} = (C - (27 - -100))^2 = (0-127)^2, (127-127)^2
    ids, dd, *_ = oracle.query(np.array([27], np.int8), s, 1, 3)
    assert ids.tolist() == [1, 0, 2] and dd.tolist() == [0, 127 * 127, 127 * 127]


# ---------------------------------------------------------------- closed forms / library routines

def _random_snapshot(rng, N=300, D=8, nlist=6, L=64, M=4, Ks=8, lo=-20, hi=20):
    db = rng.integers(lo, hi + 1, size=(N, D)).astype(np.int8)
    cent = rng.choice(N, nlist, replace=False)
    code = np.stack([rng.choice(N, Ks, replace=False) for _ in range(M)])
    return db, oracle.build_snapshot(db, nlist, L, M, Ks, cent, code)


def test_step1_matches_scipy_cdist():
    """Step 1 against an independent library routine (scipy cdist,
    float64, exact for these integer magnitudes)."""
    rng = np.random.default_rng(1)
    db, s = _random_snapshot(rng, lo=-128, hi=127)
    qs = rng.integers(-128, 128, size=(20, s.D)).astype(np.int8)
    ref = cdist(qs.astype(np.float64), s.centroids.astype(np.float64), "sqeuclidean")
    for a in range(len(qs)):
        assert oracle.step1_centroid_distances(qs[a], s).tolist() == np.rint(ref[a]).astype(np.int64).tolist()
    # q == mu_3 -> d_3 = 0 (SPEC.md step1 example)
    assert oracle.step1_centroid_distances(s.centroids[3], s)[3] == 0


def test_step3_zero_case():
    """q == mu_i and C_{m,0} = 0-block -> LUT_{i,m,0} = 0."""
    s = vo.Snapshot(centroids=np.array([[3, -2, 5, 1]], np.int8),
                    codebooks=np.array([[[0, 0], [1, 1]], [[0, 0], [2, -2]]], np.int8),
                    ids=np.zeros((1, 1), np.int32), codes=np.zeros((1, 1, 2), np.uint8),
                    counts=np.ones(1, np.int32), list_of=np.zeros(1, np.int32))
    lut = oracle.step3_adc_tables(s.centroids[0], s, np.array([0]))
    assert lut[0, :, 0].tolist() == [0, 0]
    assert lut[0, :, 1].tolist() == [2, 8]


def test_adc_equals_distance_to_reconstruction():
    """Closed form: sum_m dist(C_{m,c_m}, (q - mu_i)^{(m)}) = dist(q, mu_i + xhat_{i,j}) where
    xhat is the concatenation of the selected codewords (PAPER.md:383-401 with D = Md).
    Computed independently with scipy cdist on the reconstructed vectors.  A dropped
    term, a wrong sub-block index or a transposed LUT in Steps 3-4 fails this."""
    rng = np.random.default_rng(2)
    db, s = _random_snapshot(rng, N=500, D=12, nlist=5, L=128, M=3, Ks=16, lo=-60, hi=60)
    qs = rng.integers(-128, 128, size=(10, s.D)).astype(np.int8)
    M, Ks, d = s.codebooks.shape
    for q in qs:
        _, _, probes, _, cand = oracle.query(q, s, s.nlist, 5)
        for rho, i in enumerate(probes):
            cnt = s.counts[i]
            xhat = np.concatenate([s.codebooks[m][s.codes[i, :cnt, m]] for m in range(M)], axis=1)
            recon = s.centroids[i].astype(np.float64) + xhat.astype(np.float64)
            ref = cdist(q[None].astype(np.float64), recon, "sqeuclidean")[0]
            assert cand[rho, :cnt].tolist() == np.rint(ref).astype(np.int64).tolist()
            assert (cand[rho, cnt:] == oracle.D_MAX).all()


def test_bruteforce_degeneracy_exact_knn():
    """P6 / SPEC.md:350: n_probe = n_list = 1, M = D (d = 1) and a codebook containing
    every residual value exactly -> the ADC distance is the exact squared L2 distance and
    the top-k equals exhaustive k-NN with the (dist, id) tie-break."""
    rng = np.random.default_rng(3)
    D, N, k = 6, 400, 25
    db = rng.integers(-3, 4, size=(N, D)).astype(np.int8)
    db[0] = 0                                  # centroid row 0 = all zeros
    for v in range(-3, 4):                     # rows 1..7 = constant vectors -3..3
        db[v + 4] = v
    s = oracle.build_snapshot(db, 1, N, D, 8, [0], [[1, 2, 3, 4, 5, 6, 7, 8]] * D)
    assert (s.codebooks.reshape(D, 8)[:, :7] == np.arange(-3, 4)[None, :]).all()
    for _ in range(20):
        q = rng.integers(-6, 7, size=D).astype(np.int8)
        ids, dd, *_ = oracle.query(q, s, 1, k)
        exact = ((db.astype(np.int64) - q.astype(np.int64)) ** 2).sum(1)
        order = sorted(range(N), key=lambda t: (exact[t], t))[:k]     # exhaustive k-NN
        assert ids.tolist() == order
        assert dd.tolist() == [int(exact[t]) for t in order]


def test_lowacc_shape_reduces_to_id_order():
    """Paper E2 low-acc shape has K = 1: every code is 0, so every valid
    candidate of a list has the same ADC distance and Step 5 orders by id alone."""
    rng = np.random.default_rng(4)
    N, D, nlist, L = 200, 8, 4, 64
    db = rng.integers(-50, 50, size=(N, D)).astype(np.int8)
    s = oracle.build_snapshot(db, nlist, L, 4, 1, rng.choice(N, nlist, replace=False),
                              rng.choice(N, (4, 1), replace=False))
    assert (s.codes == 0).all()
    q = rng.integers(-50, 50, size=D).astype(np.int8)
    ids, dd, probes, _, cand = oracle.query(q, s, 1, 10)
    i = probes[0]
    assert len(set(cand[0, :s.counts[i]].tolist())) == 1
    assert ids.tolist() == sorted(s.ids[i, :s.counts[i]].tolist())[:10]


# ---------------------------------------------------------------- build: brute force + replay

def _greedy_bruteforce(db, mu, L):
    """Literal B2 with the full (e, i) ranking of every vector (tiny inputs only)."""
    nlist = mu.shape[0]
    counts = [0] * nlist
    out = []
    for t in range(db.shape[0]):
        e = [oracle.dist(db[t], mu[i]) for i in range(nlist)]
        for i in sorted(range(nlist), key=lambda i: (e[i], i)):
            if counts[i] < L:
                counts[i] += 1
                out.append(i)
                break
    return out


@pytest.mark.parametrize("seed", range(6))
def test_greedy_matches_bruteforce_tiny(seed):
    rng = np.random.default_rng(100 + seed)
    N, D, nlist = 60, 3, 5
    L = int(np.ceil(N / nlist)) + seed % 3          # tight capacity -> heavy overflow
    db = rng.integers(-2, 3, size=(N, D)).astype(np.int8)   # tiny range -> many ties
    mu = db[rng.choice(N, nlist, replace=False)]
    assert vo.assign_greedy(db, mu, L, chunk=7).tolist() == _greedy_bruteforce(db, mu, L)


@pytest.mark.parametrize("seed", range(4))
def test_greedy_rowwise_matches_bruteforce_tiny(seed):
    """The vector-by-vector reference loop itself against the literal (e, i) ranking."""
    rng = np.random.default_rng(200 + seed)
    N, D, nlist = 70, 2, 6
    L = int(np.ceil(N / nlist)) + seed % 2
    db = rng.integers(-2, 3, size=(N, D)).astype(np.int8)
    mu = db[rng.choice(N, nlist, replace=False)]
    assert vo._assign_greedy_rowwise(db, mu, L).tolist() == _greedy_bruteforce(db, mu, L)


@pytest.mark.parametrize("chunk", [1, 64, 777, 4096])
@pytest.mark.parametrize("slack", [0, 3, 50])
def test_greedy_blocked_matches_rowwise(chunk, slack):
    """The chunked evaluation of B2 (lists closing mid-chunk, stale choices of the look-ahead
    workers) equals the vector-by-vector loop, with heavy overflow (slack 0: every list fills),
    many ties (a 5-value alphabet) and chunk boundaries everywhere."""
    rng = np.random.default_rng(chunk + 7 * slack)
    N, D, nlist = 6000, 3, 37
    L = int(np.ceil(N / nlist)) + slack
    db = rng.integers(-2, 3, size=(N, D)).astype(np.int8)
    db[: N // 3] = rng.integers(-60, 60, size=(N // 3, D))
    mu = db[rng.choice(N, nlist, replace=False)]
    got = vo.assign_greedy(db, mu, L, chunk=chunk)
    assert np.array_equal(got, vo._assign_greedy_rowwise(db, mu, L))
    assert np.bincount(got, minlength=nlist).max() <= L


def greedy_replay_violations(db, s, sample=None):
    """P7 replay check that does not re-run the algorithm: for vector t in list i, every
    list ranked before i by (e, i) already held L members with id < t, and list i held
    fewer than L members with id < t."""
    L = s.L
    mu = s.centroids.astype(np.int64)
    # slot ids are ascending inside a list (R7) -> members with id < t = searchsorted
    ts = range(db.shape[0]) if sample is None else sample
    bad = []
    for t in ts:
        i = int(s.list_of[t])
        e = ((db[t].astype(np.int64)[None, :] - mu) ** 2).sum(1)
        key_i = (e[i], i)
        before = [j for j in range(s.nlist) if (e[j], j) < key_i]
        for j in before:
            if np.searchsorted(s.ids[j, :s.counts[j]], t) < L:
                bad.append((t, j))
        if np.searchsorted(s.ids[i, :s.counts[i]], t) >= L:
            bad.append((t, i))
    return bad


def test_greedy_replay_property_c0_shape():
    from synth import generate, get_config
    cfg = get_config("c0").with_(L=520)              # 4096 <= 8*520: forces overflow
    inp = generate(cfg)
    s = oracle.build_snapshot(inp.db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    assert (s.counts == cfg.L).sum() >= 1
    assert greedy_replay_violations(inp.db, s) == []


def test_snapshot_structure_and_codes():
    """Fixed shape, capacity, padding content (R7), the
    codebook rule B4 and brute-force argmin codes B5 (P8)."""
    rng = np.random.default_rng(5)
    N, D, nlist, L, M, Ks = 700, 8, 6, 130, 2, 16
    db = rng.integers(-128, 128, size=(N, D)).astype(np.int8)
    cent = rng.choice(N, nlist, replace=False)
    code = np.stack([rng.choice(N, Ks, replace=False) for _ in range(M)])
    s = oracle.build_snapshot(db, nlist, L, M, Ks, cent, code)
    d = D // M
    assert s.ids.shape == (nlist, L) and s.codes.shape == (nlist, L, M)
    assert (s.counts <= L).all() and s.counts.sum() == N
    assert sorted(s.ids[s.ids >= 0].tolist()) == list(range(N))
    for i in range(nlist):
        c = s.counts[i]
        assert (np.diff(s.ids[i, :c]) > 0).all()
        assert (s.ids[i, c:] == -1).all() and (s.codes[i, c:] == 0).all()
        assert (s.list_of[s.ids[i, :c]] == i).all()
    resid = db.astype(np.int64) - s.centroids[s.list_of].astype(np.int64)
    for m in range(M):
        for c in range(Ks):
            exp = np.clip(resid[code[m][c], m * d:(m + 1) * d], -127, 127)
            assert s.codebooks[m, c].tolist() == exp.tolist()
    # brute-force argmin, first minimum on ties (R6)
    for t in range(0, N, 7):
        i = s.list_of[t]
        slot = int(np.searchsorted(s.ids[i, :s.counts[i]], t))
        for m in range(M):
            errs = [int(((resid[t, m * d:(m + 1) * d] - s.codebooks[m, c].astype(np.int64)) ** 2).sum())
                    for c in range(Ks)]
            assert s.codes[i, slot, m] == errs.index(min(errs))


def test_build_errors():
    db = np.zeros((10, 4), np.int8)
    with pytest.raises(ValueError):
        oracle.build_snapshot(db, 2, 4, 2, 2, [0, 1], [[0, 1], [2, 3]])       # N > nlist*L
    with pytest.raises(ValueError):
        oracle.build_snapshot(db, 2, 8, 2, 2, [0, 0], [[0, 1], [2, 3]])       # duplicate centroid rows
    with pytest.raises(ValueError):
        oracle.build_snapshot(db, 2, 8, 3, 2, [0, 1], [[0, 1], [2, 3], [4, 5]])  # D % M != 0


# ---------------------------------------------------------------- prover witness (NEXT-2)

def test_witness_consistent_with_pinned_steps():
    """The witness against the already-pinned steps and the paper's own checks:
    S^sorted_{idx,dist} is a permutation of [n_list] in nondecreasing d whose first n_probe entries
    are Step 2's P(q); every selected entry equals dist(C_{m,code}, (q-mu_i)^(m))
    recomputed by brute force and the entries of a valid slot sum to its Step-4 distance (the
    multiset-inclusion statement of PAPER.md:640-648); S^sorted_{item,dist} is the multiset of
    S^orig in nondecreasing D whose first k pairs are Step 5's output."""
    rng = np.random.default_rng(21)
    db, s = _random_snapshot(rng, N=400, D=8, nlist=7, L=80, M=4, Ks=8, lo=-40, hi=40)
    M, Ks, d = s.codebooks.shape
    for _ in range(6):
        q = rng.integers(-128, 128, size=s.D).astype(np.int8)
        nprobe, k = int(rng.integers(1, s.nlist + 1)), int(rng.integers(1, 30))
        order, od, ell, items, dists = oracle.witness(q, s, nprobe)
        ids, dd, probes, dP, cand = oracle.query(q, s, nprobe, k)
        assert sorted(order.tolist()) == list(range(s.nlist)) and (np.diff(od) >= 0).all()
        assert order[:nprobe].tolist() == probes.tolist()
        assert od.tolist() == [oracle.dist(q, s.centroids[i]) for i in order]
        for rho, i in enumerate(probes):
            res = q.astype(np.int64) - s.centroids[i].astype(np.int64)
            for j in range(0, s.L, 9):
                for m in range(M):
                    c = int(s.codes[i, j, m])
                    assert ell[rho, j, m] == oracle.dist(s.codebooks[m, c], res[m * d:(m + 1) * d])
                if s.ids[i, j] != -1:
                    assert ell[rho, j].sum() == cand[rho, j]
        orig = sorted(zip(s.ids[probes].reshape(-1).tolist(), cand.reshape(-1).tolist()))
        assert sorted(zip(items.tolist(), dists.tolist())) == orig and (np.diff(dists) >= 0).all()
        assert items[:k].tolist() == ids.tolist() and dists[:k].tolist() == dd.tolist()


# ---------------------------------------------------------------- Alg. 1 rebalancing (NEXT-3)

@pytest.mark.parametrize("db,rows,L,expect,rounds", [
    ([3, 2, 1, 0, 10, 11, 20], [3, 4, 6], 3, [1, 0, 0, 0, 1, 1, 2], 1),
    ([0, 1, 2, 3, 4, 10, 11, 30], [0, 5, 7], 3, [0, 0, 0, 2, 1, 1, 1, 2], 2),
])
def test_rebalance_hand_examples(db, rows, L, expect, rounds):
    """Alg. 1 on the two 1-D cases derived by hand in
    tests/golden/rebalance_example.md."""
    x = np.array(db, np.int8)[:, None]
    got, r = vo.assign_rebalance(x, x[rows], L, return_rounds=True)
    assert got.tolist() == expect and r == rounds


def test_rebalance_invariants_and_no_op():
    """Alg. 1 ensures |X_i| <= n, conserves the vectors, leaves an assignment with no
    overfull list unchanged (the while loop does not run), and only moves vectors out of lists that
    were overfull in the initial assignment."""
    rng = np.random.default_rng(31)
    for trial in range(20):
        N, D, nlist = int(rng.integers(20, 200)), int(rng.integers(1, 5)), int(rng.integers(2, 9))
        L = int(np.ceil(N / nlist)) + int(rng.integers(0, 3))
        db = rng.integers(-6, 7, size=(N, D)).astype(np.int8)
        mu = db[rng.choice(N, nlist, replace=False)]
        init = vo.nearest_lists(db, mu)
        got = vo.assign_rebalance(db, mu, L)
        counts0 = np.bincount(init, minlength=nlist)
        assert (np.bincount(got, minlength=nlist) <= L).all()
        moved = got != init
        assert (counts0[init[moved]] > L).all()
        if (counts0 <= L).all():
            assert not moved.any()


# ---------------------------------------------------------------- 16-bit fixed point (NEXT-1)

def test_fixed_point_encoding_by_hand():
    """v -> round((2^16 - 1) v / v_max); worked by hand with v_max = 4:
    4 -> 65535, -4 -> -65535, 1 -> 16383.75 -> 16384, -1 -> -16384, 0 -> 0,
    2/65535*4... the half case 4 * 0.5 / 65535 -> 0.5 -> 1 (half away from zero, R18)."""
    x = np.array([4.0, -4.0, 1.0, -1.0, 0.0, 2.0 / 65535.0, -2.0 / 65535.0])
    got = oracle.encode_fixed_point(x, 4.0)
    assert got.tolist() == [65535, -65535, 16384, -16384, 0, 1, -1]
    assert got.dtype == np.int32


def test_fixed_point_rounding_just_below_half():
    """PAPER.md:781-782's rounding at the representable neighbours of the half-integers (R18:
    half away from zero).  With v_max = 65535 the scaled value is y = v exactly, so v = the largest
    double below 0.5 must round to 0 (an implementation computing floor(y + 0.5) returns 1: the
    sum rounds to 1.0), the smallest double above 0.5 to 1, 2.5 to 3, nextafter(2.5, 0) to 2,
    and every case mirrored for negative v."""
    below, above = np.nextafter(0.5, 0.0), np.nextafter(0.5, 1.0)
    v = np.array([below, above, 0.5, 2.5, np.nextafter(2.5, 0.0), np.nextafter(1.5, 2.0), 1.0, 0.0])
    exp = [0, 1, 1, 3, 2, 2, 1, 0]
    assert oracle.encode_fixed_point(v, 65535.0).tolist() == exp
    assert oracle.encode_fixed_point(-v, 65535.0).tolist() == [-e for e in exp]
    # the same through float32 input (the C ABI takes float32): 0.5 - 2^-25 is a float32 value
    x32 = np.array([np.nextafter(np.float32(0.5), np.float32(0))], dtype=np.float32)
    assert oracle.encode_fixed_point(x32, 65535.0).tolist() == [0]
    assert oracle.encode_fixed_point(-x32, 65535.0).tolist() == [0]


def test_fixed_point_variant_equals_int8_semantics_when_nothing_saturates():
    """Special case reducing to the pinned int8 path: on int8-valued data whose residuals never
    leave [-127, 127] (so R5's saturation is a no-op), the fixed-point oracle (int32 storage, int64
    distances, unsaturated codewords R19) must return exactly the int8 oracle's snapshot and
    query results -- only the storage width differs."""
    rng = np.random.default_rng(41)
    N, D, nlist, L, M, Ks = 500, 8, 6, 120, 4, 16
    db8 = rng.integers(-60, 61, size=(N, D)).astype(np.int8)
    cent = rng.choice(N, nlist, replace=False)
    code = np.stack([rng.choice(N, Ks, replace=False) for _ in range(M)])
    s8 = oracle.build_snapshot(db8, nlist, L, M, Ks, cent, code)
    s32 = oracle.build_snapshot(db8.astype(np.int32), nlist, L, M, Ks, cent, code)
    assert s32.fx and not s8.fx
    for name in ("centroids", "codebooks", "ids", "codes", "counts", "list_of"):
        assert np.array_equal(getattr(s8, name).astype(np.int64), getattr(s32, name).astype(np.int64)), name
    qs = rng.integers(-60, 61, size=(12, D)).astype(np.int8)
    r8 = oracle.query_batch(s8, qs, 3, 20)
    r32 = oracle.query_batch(s32, qs.astype(np.int32), 3, 20)
    for key in r8:
        a, b = r8[key].astype(np.int64), r32[key].astype(np.int64)
        if key == "trace_cand_dist":   # padding: d_max differs (2^31 - 1 vs 2^63 - 1)
            a = np.where(a == oracle.D_MAX, -1, a)
            b = np.where(b == oracle.D_MAX_FX, -1, b)
        assert np.array_equal(a, b), key


def test_fixed_point_adc_is_distance_to_reconstruction():
    """Closed form at 17-bit magnitudes (int64 arithmetic): every valid candidate distance equals
    dist(q, mu_i + xhat) computed independently with Python integers."""
    rng = np.random.default_rng(42)
    x = rng.standard_normal((300, 8))
    q = rng.standard_normal((4, 8))
    v_max = float(max(np.abs(x).max(), np.abs(q).max()))
    db = oracle.encode_fixed_point(x, v_max)
    qq = oracle.encode_fixed_point(q, v_max)
    s = oracle.build_snapshot(db, 5, 80, 2, 16, rng.choice(300, 5, replace=False),
                              np.stack([rng.choice(300, 16, replace=False) for _ in range(2)]))
    assert s.fx and np.abs(s.codebooks).max() > 127            # genuinely beyond int8
    for qv in qq:
        _, _, probes, _, cand = oracle.query(qv, s, 5, 10)
        for rho, i in enumerate(probes):
            for j in range(0, s.counts[i], 7):
                xhat = [int(s.codebooks[m, s.codes[i, j, m], u]) for m in range(2) for u in range(4)]
                ref = sum((int(qv[u]) - int(s.centroids[i, u]) - xhat[u]) ** 2 for u in range(8))
                assert cand[rho, j] == ref
