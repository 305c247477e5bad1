"""Property tests of the oracle on random tiny instances (SPEC.md:354-359 invariants,
PAPER.md partial-order conditions of Steps 2 and 5)."""
import numpy as np
from hypothesis import given, settings, strategies as st

import oracle


@st.composite
def instances(draw):
    D_over_M = draw(st.integers(1, 3))
    M = draw(st.integers(1, 4))
    D = D_over_M * M
    nlist = draw(st.integers(1, 6))
    L = draw(st.integers(1, 12))
    N = draw(st.integers(max(nlist, 1), nlist * L))
    Ks = draw(st.integers(1, min(N, 8)))
    span = draw(st.sampled_from([1, 3, 40, 127]))
    seed = draw(st.integers(0, 2**31 - 1))
    rng = np.random.default_rng(seed)
    db = rng.integers(-span, span + 1, size=(N, D)).astype(np.int8)
    cent = rng.choice(N, nlist, replace=False)
    code = np.stack([rng.choice(N, Ks, replace=False) for _ in range(M)])
    s = oracle.build_snapshot(db, nlist, L, M, Ks, cent, code)
    nprobe = draw(st.integers(1, nlist))
    k = draw(st.integers(1, nprobe * L))
    q = rng.integers(-128, 128, size=D).astype(np.int8)
    return db, s, q, nprobe, k


@settings(max_examples=300, deadline=None)
@given(instances())
def test_query_invariants(inst):
    db, s, q, nprobe, k = inst
    ids, dd, probes, dP, cand = oracle.query(q, s, nprobe, k)
    d = oracle.step1_centroid_distances(q, s)
    # Step 2 partial order and distinctness
    assert len(set(probes.tolist())) == nprobe
    assert (np.diff(d[probes]) >= 0).all()
    rest = np.setdiff1d(np.arange(s.nlist), probes)
    if len(rest):
        assert d[probes[-1]] <= d[rest].min()
    assert dP.tolist() == d[probes].tolist()
    # scan budget: exactly N_sel candidate scores
    assert cand.shape == (nprobe, s.L)
    # Step 5 partial order + permutation soundness
    all_items = s.ids[probes].reshape(-1)
    all_d = cand.reshape(-1)
    assert (np.diff(dd) >= 0).all()
    assert dd[-1] <= np.sort(all_d)[k - 1] if k < len(all_d) else True
    pairs = sorted(zip(all_d.tolist(), all_items.tolist()))
    assert list(zip(dd.tolist(), ids.tolist())) == pairs[:k]
    # padding never returned when >= k valid candidates exist (R11)
    n_valid = int((all_items >= 0).sum())
    if n_valid >= k:
        assert (ids >= 0).all() and (dd < oracle.D_MAX).all()
    else:
        assert (ids[n_valid:] == -1).all() and (dd[n_valid:] == oracle.D_MAX).all()
    # masking
    assert ((cand == oracle.D_MAX) == (s.ids[probes] == -1)).all()
    # determinism
    ids2, dd2, *_ = oracle.query(q, s, nprobe, k)
    assert ids2.tolist() == ids.tolist() and dd2.tolist() == dd.tolist()


@settings(max_examples=150, deadline=None)
@given(instances())
def test_build_invariants(inst):
    db, s, *_ = inst
    N = db.shape[0]
    assert (s.counts <= s.L).all() and int(s.counts.sum()) == N
    assert sorted(s.ids[s.ids >= 0].tolist()) == list(range(N))
    for i in range(s.nlist):
        c = s.counts[i]
        assert (np.diff(s.ids[i, :c]) > 0).all()
        assert (s.ids[i, c:] == -1).all()
