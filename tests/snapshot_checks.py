"""Checks of a fixed-shape IVF-PQ snapshot against the build rules themselves (SURVEY.md §8(c)
B1-B6, pins P7/P8) -- test infrastructure, used where the oracle's own build is too slow."""
import numpy as np


def check_snapshot(cfg, inp, snap, rng, n_replay=150, n_slots=400, fx=False):
    """B1-B6 checked against the rules themselves (not against a second implementation).
    fx: the 16-bit fixed-point variant (int32 coordinates, unsaturated codewords, R18/R19)."""
    db = inp.db
    N, D = db.shape
    L, M = cfg.L, cfg.M
    d = D // M
    ids, codes, counts, mu, cb, list_of = (snap[k] for k in ("ids", "codes", "counts", "centroids", "codebooks",
                                                             "list_of"))
    # B1: centroids are the sampled rows
    assert np.array_equal(mu, db[inp.centroid_rows])
    # B6 / R7: fixed shape, capacity, valid prefix in ascending id, padding (-1, code 0), a permutation
    assert (counts <= L).all() and counts.sum() == N
    slot = np.arange(L)[None, :]
    valid = slot < counts[:, None]
    assert (ids[~valid] == -1).all() and (codes[~valid] == 0).all()
    assert np.array_equal(np.sort(ids[valid]), np.arange(N))
    v_ids = np.where(valid, ids, np.iinfo(np.int32).max)
    assert (np.diff(v_ids, axis=1)[valid[:, 1:]] > 0).all()
    rows, cols = np.nonzero(valid)
    assert np.array_equal(list_of[ids[rows, cols]], rows)
    # B3/B4 (R4, R5): codewords = saturated residual sub-vectors of the sampled rows (final lists)
    cw = inp.codeword_rows
    for m in range(M):
        r = db[cw[m], m * d:(m + 1) * d].astype(np.int64) - mu[list_of[cw[m]], m * d:(m + 1) * d].astype(np.int64)
        exp = r.astype(np.int32) if fx else np.clip(r, -127, 127).astype(np.int8)
        assert cb.dtype == exp.dtype and np.array_equal(cb[m], exp), m
    # B2 (R1, R2) replayed for sampled vectors: every list ranked before t's list by (e, i) already
    # held L members with id < t, and t's list held fewer than L
    mu64 = mu.astype(np.int64)
    ts = np.unique(np.concatenate([rng.choice(N, n_replay, replace=False), [0, N - 1]]))
    for t in ts:
        i = int(list_of[t])
        e = ((db[t].astype(np.int64)[None, :] - mu64) ** 2).sum(1)
        before = np.nonzero((e < e[i]) | ((e == e[i]) & (np.arange(len(e)) < i)))[0]
        for j in before:
            assert np.searchsorted(ids[j, :counts[j]], t) >= L, (t, j)
        assert np.searchsorted(ids[i, :counts[i]], t) < L, t
    # B5 (R6): codes of sampled valid slots = brute-force argmin, lowest codeword on ties
    pick = rng.choice(len(rows), min(n_slots, len(rows)), replace=False)
    cb64 = cb.astype(np.int64)
    for a in pick:
        i, j = rows[a], cols[a]
        res = db[ids[i, j]].astype(np.int64) - mu64[i]
        for m in range(M):
            err = ((res[m * d:(m + 1) * d][None, :] - cb64[m]) ** 2).sum(1)
            assert codes[i, j, m] == int(np.argmin(err)), (i, j, m)
