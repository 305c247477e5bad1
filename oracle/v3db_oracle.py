"""V3DB fixed-shape IVF-PQ oracle -- TEST INFRASTRUCTURE ONLY.

Plain numpy, int64 arithmetic, following the paper step by step:
  * build:  PAPER.md:93-100 (IVF + PQ of residuals), :288-294 (capacity bound n,
    padding with validity flag), :331-340 (snapshot contents), with BASELINE.json's
    shaping rule (nearest centroid, lowest index on ties, overflow to the
    next-nearest list with room) in place of Alg. 1 -- SURVEY.md §8(c) B1-B6, R1-R8.
  * query:  PAPER.md:351-428, §4.2 Steps 1-5.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this module.  It shares no code with the CUDA path and imports
nothing from it.  Every function below is pinned by tests in tests/test_oracle_*.py
(see DESIGN.md "Oracle pins"); none is "parity unpinned".

Readings where the paper is silent (binding on oracle and library alike; DESIGN.md
lists them): R2 ranking key (e, i); R4 residual w.r.t. the final list; R5 codewords
saturated to [-127,127], residuals not clamped; R6 encode ties -> lowest codeword;
R7 valid slots first in ascending id, padding id -1 / code 0; R8 d_max = 2^31-1;
R9/R10 total orders (d_i, i) and (D, id); R11 < k valid -> (-1, d_max) fill;
R12 flatten S^orig in probe-rank order then slot order.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

# R8: "a public constant d_max that exceeds any attainable d~".
D_MAX = 2**31 - 1
# The 16-bit fixed-point variant (NEXT-1) has int64 distances: d_max = 2^63 - 1.
D_MAX_FX = 2**63 - 1
FX_SCALE = 2**16 - 1


def encode_fixed_point(x, v_max: float):
    """each coordinate v becomes round((2^16 - 1) * v / v_max), v_max the largest
    |coordinate| over all involved vectors.  Reading R18: the product and quotient in IEEE double
    (in that order), round half away from zero.  Returns int32 in [-(2^16-1), 2^16-1]."""
    y = np.asarray(x, dtype=np.float64) * float(FX_SCALE) / float(v_max)
    # round half away from zero on |y|: floor(|y|) plus one when the fractional part is >= 1/2.
    # |y| - floor(|y|) is exact in IEEE double, so the comparison is the mathematical one
    # (floor(|y| + 0.5) would round y = nextafter(0.5, 0) up: the addition rounds to 1.0).
    a = np.abs(y)
    f = np.floor(a)
    r = np.sign(y) * (f + (a - f >= 0.5))
    assert np.abs(r).max(initial=0) <= FX_SCALE
    return r.astype(np.int32)


def dist(x, y) -> int:
    """dist(x, y) := sum_t (x_t - y_t)^2  (§4.2), exact over the integers."""
    x = np.asarray(x, dtype=np.int64)
    y = np.asarray(y, dtype=np.int64)
    return int(((x - y) ** 2).sum())


@dataclass
class Snapshot:
    """Fixed-shape snapshot: centroids mu, PQ codebooks C_{m,c},
    and per (list i, slot j) the record (f_ij, item_ij, v^PQ_ij) with f = (id != -1)."""
    centroids: np.ndarray   # int8  [nlist][D]          mu_i
    codebooks: np.ndarray   # int8  [M][Ks][d]          C_{m,c}
    ids: np.ndarray         # int32 [nlist][L]          item_{i,j}; -1 = padding (f_{i,j} = 0)
    codes: np.ndarray       # uint8 [nlist][L][M]       v^{(m)}_{i,j}
    counts: np.ndarray      # int32 [nlist]             number of valid slots
    list_of: np.ndarray     # int32 [N]                 final list of each vector

    @property
    def nlist(self): return self.ids.shape[0]
    @property
    def L(self): return self.ids.shape[1]
    @property
    def M(self): return self.codebooks.shape[0]
    @property
    def Ks(self): return self.codebooks.shape[1]
    @property
    def D(self): return self.centroids.shape[1]
    @property
    def fx(self):
        """16-bit fixed-point variant (NEXT-1): int32 coordinates, int64 distances."""
        return self.centroids.dtype == np.int32
    @property
    def d_max(self): return D_MAX_FX if self.fx else D_MAX


# ----------------------------------------------------------------------------------------
# Build (offline index shaping)
# ----------------------------------------------------------------------------------------

def _rank_keys(x: np.ndarray, mu: np.ndarray) -> np.ndarray:
    """key_{t,i} = ||mu_i||^2 - 2 <x_t, mu_i> = e_{t,i} - ||x_t||^2, exact.

    For a fixed vector t, ordering the lists by e_{t,i} is the same as ordering them by
    key_{t,i} (they differ by the per-t constant ||x_t||^2), so the ranking of B2 can
    use key.  One library matmul of the augmented rows [x_t, 1] . [-2 mu_i, ||mu_i||^2]
    gives key directly; it runs in float32 when every partial sum is an integer below 2^24
    (exact), else in float64 (exact below 2^53)."""
    mun = (mu.astype(np.int64) ** 2).sum(1)
    amax = int(max(np.abs(x).max(initial=0), np.abs(mu).max(initial=0), 1))
    bound = int(mun.max(initial=0)) + 2 * amax * amax * x.shape[1] + 1
    assert bound < 2**53
    ft = np.float32 if bound < 2**24 else np.float64
    xa = np.empty((x.shape[0], x.shape[1] + 1), ft)
    xa[:, :-1] = x
    xa[:, -1] = 1
    ma = np.empty((mu.shape[0], mu.shape[1] + 1), ft)
    ma[:, :-1] = -2 * mu.astype(np.int64)
    ma[:, -1] = mun
    return xa @ ma.T


def assign_greedy(db: np.ndarray, mu: np.ndarray, L: int, chunk: int = 4096) -> np.ndarray:
    """B2: streaming greedy assignment with capacity L (BASELINE.json shaping rule, R1/R2).

    For t = 0, 1, ..., N-1 in order: rank the lists by (e_{t,i} = dist(db[t], mu_i), i)
    ascending and append t to the FIRST list in that ranking whose current count is < L.
    The first list in the (e, i) ranking that has room is exactly the lowest-index
    minimiser of e over the lists that have room (np.argmin returns the first minimum).

    Evaluation order (the same result as the vector-by-vector loop, pinned against it in
    tests/test_oracle_pins.py): within a chunk of vectors every vector first takes the minimiser
    over the lists that have room at the chunk's start.  That is the sequential choice for every
    vector up to the first one whose chosen list its predecessors in the chunk have filled (a list
    that fills up is never the choice of a vector before that point, so removing it from the lists
    with room changes no earlier choice).  The vectors before that point are placed at once, the
    lists that became full are closed, the choices that pointed at them are recomputed over the
    remaining lists, and the walk resumes at that vector.  A thread pool computes the ranking keys
    and first choices of chunks ahead, against the lists that had room when it started: a list
    only ever fills up, so such a choice is still the minimiser over the lists with room at
    placement time unless it has filled meanwhile -- and those choices are recomputed.
    """
    from concurrent.futures import ThreadPoolExecutor

    N = db.shape[0]
    nlist = mu.shape[0]
    list_of = np.empty(N, dtype=np.int32)
    counts = np.zeros(nlist, dtype=np.int64)
    closed = np.zeros(nlist, dtype=bool)               # lists that are full

    def rank(lo, closed_then):
        e = _rank_keys(db[lo:min(N, lo + chunk)], mu)    # [chunk, nlist] e_{t,i} - ||x_t||^2
        e += np.where(closed_then, np.inf, 0).astype(e.dtype)   # only lists with room (as of closed_then)
        return e, np.argmin(e, axis=1)                 # nearest list with room, lowest index on ties

    starts = list(range(0, N, chunk))
    ahead = max(2, min(16, (os.cpu_count() or 4)))
    with ThreadPoolExecutor(max_workers=ahead) as ex:
        futs = [ex.submit(rank, lo, closed.copy()) for lo in starts[:ahead]]
        for c, lo in enumerate(starts):
            e, choice = futs[c].result()
            futs[c] = None
            room = np.where(closed, np.inf, 0).astype(e.dtype)
            n = e.shape[0]
            redo = np.flatnonzero(closed[choice])       # choices that filled since the worker started
            if len(redo):
                choice[redo] = np.argmin(e[redo] + room, axis=1)
            pos = 0
            while pos < n:
                ch = choice[pos:]
                # ordinal of each vector among the vectors of ch that chose the same list
                order = np.argsort(ch, kind="stable")
                srt = ch[order]
                first = np.r_[0, np.flatnonzero(srt[1:] != srt[:-1]) + 1]
                run = np.diff(np.r_[first, len(srt)])
                ordinal = np.empty(len(ch), dtype=np.int64)
                ordinal[order] = np.arange(len(srt)) - np.repeat(first, run)
                over = counts[ch] + ordinal >= L            # its list is full when its turn comes
                b = int(np.argmax(over)) if over.any() else len(ch)
                list_of[lo + pos:lo + pos + b] = ch[:b]
                counts += np.bincount(ch[:b], minlength=nlist)
                pos += b
                if pos == n:
                    break
                closed |= counts >= L                       # close the lists that filled up
                room[closed] = np.inf
                redo = np.flatnonzero(closed[choice[pos:]]) + pos
                choice[redo] = np.argmin(e[redo] + room, axis=1)
                assert not closed[choice[pos]], "N > nlist * L (infeasible)"
            closed |= counts >= L
            if c + ahead < len(starts):
                futs.append(ex.submit(rank, starts[c + ahead], closed.copy()))
    return list_of


def _assign_greedy_rowwise(db: np.ndarray, mu: np.ndarray, L: int) -> np.ndarray:
    """B2 vector by vector (the definition's loop), for the pins of assign_greedy."""
    N, nlist = db.shape[0], mu.shape[0]
    e = _rank_keys(db, mu)
    counts = np.zeros(nlist, dtype=np.int64)
    room = np.zeros(nlist, dtype=e.dtype)
    out = np.empty(N, dtype=np.int32)
    for t in range(N):
        i = int(np.argmin(e[t] + room))
        assert counts[i] < L, "N > nlist * L (infeasible)"
        out[t] = i
        counts[i] += 1
        if counts[i] == L:
            room[i] = np.inf
    return out


def nearest_lists(db: np.ndarray, mu: np.ndarray, chunk: int = 4096) -> np.ndarray:
    """argmin_i (dist(db[t], mu_i), i) for every t: the initial assignment (R2)."""
    out = np.empty(db.shape[0], dtype=np.int64)
    for lo in range(0, db.shape[0], chunk):
        out[lo:lo + chunk] = np.argmin(_rank_keys(db[lo:lo + chunk], mu), axis=1)
    return out


def assign_rebalance(db: np.ndarray, mu: np.ndarray, L: int, return_rounds: bool = False):
    """Alg. 1 ("Capacity-constrained cluster rebalancing"), literally, on the
    nearest-centroid assignment.  Readings (R17): t* ties -> lowest list index; "sort M
    by increasing Delta" is a stable sort of M built in (cluster i ascending, v ascending) order, so
    ties keep that order.  Returns list_of (and the number of rounds)."""
    N = db.shape[0]
    nlist = mu.shape[0]
    assert N <= nlist * L, "infeasible: N > nlist * L"
    list_of = nearest_lists(db, mu)
    counts = np.bincount(list_of, minlength=nlist)
    rounds = 0
    while (counts > L).any():                                   # while exists i with n_i > n
        rounds += 1
        O = np.nonzero(counts > L)[0]                           # overfull clusters
        F = np.nonzero(counts < L)[0]                           # free clusters
        vs = np.concatenate([np.nonzero(list_of == i)[0] for i in O])   # (i ascending, v ascending)
        src = list_of[vs]
        key_f = _rank_keys(db[vs], mu[F])                       # dist(v, mu_t) - ||v||^2, t in F
        tpos = np.argmin(key_f, axis=1)                         # lowest t on ties (F ascending)
        tstar = F[tpos]
        e_t = np.rint(key_f[np.arange(len(vs)), tpos]).astype(np.int64)
        mun = (mu.astype(np.int64) ** 2).sum(1)
        e_i = mun[src] - 2 * (db[vs].astype(np.int64) * mu[src].astype(np.int64)).sum(1)
        delta = e_t - e_i                                        # Delta(v, i) (the ||v||^2 terms cancel)
        order = np.argsort(delta, kind="stable")                 # sort M by increasing Delta
        for a in order.tolist():                                 # apply the guarded moves in order
            v, i, t = int(vs[a]), int(src[a]), int(tstar[a])
            if counts[i] > L and counts[t] < L and list_of[v] == i:
                list_of[v] = t
                counts[i] -= 1
                counts[t] += 1
    return (list_of.astype(np.int32), rounds) if return_rounds else list_of.astype(np.int32)


def encode(residuals: np.ndarray, codebooks: np.ndarray, chunk: int = 65536) -> np.ndarray:
    """B5: code_t[m] = argmin_c sum_u (r_t[m d + u] - C_{m,c,u})^2, lowest c on ties (R6).

    PQ encoding of residuals.  For a fixed t the ranking of
    sum_u (r_u - C_u)^2 over c equals the ranking of ||C_c||^2 - 2 <r, C_c> (they differ by
    the per-t constant ||r||^2); those keys are integers below 2^24 (d <= 16, |r| <= 255,
    |C| <= 127), so the float32 matmul computing them is exact.  Subspaces are independent
    and run on a thread pool (numpy releases the GIL in matmul/argmin).
    """
    from concurrent.futures import ThreadPoolExecutor

    N, D = residuals.shape
    M, Ks, d = codebooks.shape
    rmax = int(max(np.abs(residuals).max(initial=0), 1))
    cmax = int(max(np.abs(codebooks).max(initial=0), 1))
    bound = d * (cmax * cmax + 2 * rmax * cmax)
    assert bound < 2**53
    ft = np.float32 if bound < 2**24 else np.float64       # exact either way
    codes = np.empty((N, M), dtype=np.uint8)

    def one(m):
        C = codebooks[m].astype(ft)                        # [Ks, d]
        cn = (C * C).sum(1)
        for lo in range(0, N, chunk):
            hi = min(N, lo + chunk)
            key = cn[None, :] - ft(2) * (residuals[lo:hi, m * d:(m + 1) * d].astype(ft) @ C.T)
            codes[lo:hi, m] = np.argmin(key, axis=1)       # lowest c on ties (R6)

    with ThreadPoolExecutor(max_workers=min(M, os.cpu_count() or 1)) as ex:
        list(ex.map(one, range(M)))
    return codes


def build_snapshot(db, nlist: int, L: int, M: int, Ks: int, centroid_rows, codeword_rows,
                   rule: str = "greedy") -> Snapshot:
    """Index shaping B1-B6.  `rule` selects
    B2: "greedy" (BASELINE.json's streaming overflow rule, R1) or "rebalance" (the paper's Alg. 1,
    PAPER.md:296-325, on the nearest-centroid assignment).  An int8 db is BASELINE.json's int8
    path; an int32 db is the 16-bit fixed-point variant (NEXT-1), whose
    codewords are the residual sub-vectors themselves (R19: no saturation; int32)."""
    fx = np.asarray(db).dtype == np.int32
    db = np.ascontiguousarray(db, dtype=np.int32 if fx else np.int8)
    N, D = db.shape
    centroid_rows = np.asarray(centroid_rows, dtype=np.int64)
    codeword_rows = np.asarray(codeword_rows, dtype=np.int64).reshape(M, Ks)
    if D % M:
        raise ValueError("D must be a multiple of M (PAPER.md:331, D = Md)")
    if not 1 <= Ks <= 256:
        raise ValueError("Ks must be in [1, 256] (1-byte codes)")
    if N > nlist * L:
        raise ValueError("infeasible: N > nlist * L (PAPER.md:290 needs |X_i| <= n)")
    if len(set(centroid_rows.tolist())) != nlist or centroid_rows.min() < 0 or centroid_rows.max() >= N:
        raise ValueError("centroid_rows must be nlist distinct rows in [0, N)")
    for m in range(M):
        if len(set(codeword_rows[m].tolist())) != Ks or codeword_rows[m].min() < 0 or codeword_rows[m].max() >= N:
            raise ValueError("codeword_rows[m] must be Ks distinct rows in [0, N)")
    d = D // M

    # B1: mu_i = db[centroid_rows[i]]  (BASELINE.json: "nlist coarse centroids = seeded-sampled database vectors")
    mu = db[centroid_rows].copy()

    # B2: nearest list, lowest index on ties, overflow to the next-nearest list with room (R1, R2)
    if rule == "greedy":
        list_of = assign_greedy(db, mu, L)
    elif rule == "rebalance":
        list_of = assign_rebalance(db, mu, L)
    else:
        raise ValueError(f"unknown shaping rule {rule!r}")

    # B3: residual r_t = db[t] - mu_{list_of[t]}, not clamped (R4, R5): int16 in [-255, 255] (int8
    # path) or int64 in [-131070, 131070] (fixed point)
    resid = db.astype(np.int64 if fx else np.int16) - mu[list_of].astype(np.int64 if fx else np.int16)

    # B4: C_{m,c} = sat_[-127,127]( r_{codeword_rows[m][c]}^{(m)} )  (R5); fixed point: no saturation (R19)
    cb = np.empty((M, Ks, d), dtype=np.int32 if fx else np.int8)
    for m in range(M):
        sub = resid[codeword_rows[m], m * d:(m + 1) * d]
        cb[m] = sub.astype(np.int32) if fx else np.clip(sub, -127, 127).astype(np.int8)

    # B5: PQ codes of the residuals
    code = encode(resid, cb)

    # B6: list i holds its members in ascending t in slots 0..count_i-1; padding (id -1, code 0) after (R7)
    ids = np.full((nlist, L), -1, dtype=np.int32)
    codes = np.zeros((nlist, L, M), dtype=np.uint8)
    counts = np.bincount(list_of, minlength=nlist).astype(np.int32)
    order = np.argsort(list_of, kind="stable")             # ascending t within each list
    start = 0
    for i in range(nlist):
        members = order[start:start + counts[i]]
        start += counts[i]
        ids[i, :counts[i]] = members
        codes[i, :counts[i]] = code[members]
    return Snapshot(mu, cb, ids, codes, counts, list_of)


# ----------------------------------------------------------------------------------------
# Query: the five-step fixed-shape semantics (§4.2)
# ----------------------------------------------------------------------------------------

def step1_centroid_distances(q, s: Snapshot) -> np.ndarray:
    """Step 1: d_i := dist(q, mu_i) for i in [n_list]."""
    q = np.asarray(q, dtype=np.int64)
    d = ((q[None, :] - s.centroids.astype(np.int64)) ** 2).sum(axis=1)
    assert d.max(initial=0) < (2**47 if s.fx else 2**31)
    return d


def step2_probe_select(d: np.ndarray, nprobe: int) -> np.ndarray:
    """Step 2: sort S^orig_{idx,dist} by distance; P(q) = first n_probe
    indices.  Ties are totalised by the list index (R9), i.e. the key is (d_i, i)."""
    nlist = d.shape[0]
    assert 1 <= nprobe <= nlist
    order = np.lexsort((np.arange(nlist), d))              # primary key d, secondary i
    return order[:nprobe]


def step3_adc_tables(q, s: Snapshot, probes: np.ndarray) -> np.ndarray:
    """Step 3: for each probed i, LUT_{i,m,c} := dist(C_{m,c}, (q - mu_i)^{(m)}).

    Returns int64 [nprobe][M][Ks] in probe-rank order."""
    q = np.asarray(q, dtype=np.int64)
    M, Ks, d = s.codebooks.shape
    C = s.codebooks.astype(np.int64)                       # [M, Ks, d]
    lut = np.empty((len(probes), M, Ks), dtype=np.int64)
    for rho, i in enumerate(probes):
        res = q - s.centroids[i].astype(np.int64)          # residual query q - mu_i
        blocks = res.reshape(M, 1, d)                      # (q - mu_i)^{(m)}
        lut[rho] = ((C - blocks) ** 2).sum(axis=2)
    return lut


def step4_candidate_distances(s: Snapshot, probes: np.ndarray, lut: np.ndarray) -> np.ndarray:
    """Step 4: d~_{i,j} := sum_m LUT_{i,m,v^{(m)}_{i,j}} and the masked
    D_{i,j} := f_ij * d~_ij + (1 - f_ij) * d_max.  Returns int64 [nprobe][L] (R12 order)."""
    M = s.M
    m_idx = np.arange(M)[None, :]
    out = np.empty((len(probes), s.L), dtype=np.int64)
    for rho, i in enumerate(probes):
        f = (s.ids[i] != -1).astype(np.int64)              # validity flag f_{i,j}
        dtil = lut[rho][m_idx, s.codes[i].astype(np.int64)].sum(axis=1)
        assert (dtil[f == 1] < s.d_max).all(), "d_max must exceed every valid d~ (PAPER.md:398-401)"
        out[rho] = np.where(f == 1, dtil, s.d_max)
    return out


def step5_topk(items: np.ndarray, dists: np.ndarray, k: int):
    """Step 5: sort S^orig_{item,dist} by distance and output the first k.
    Ties are totalised by the item id as a signed integer (R10)."""
    assert 1 <= k <= len(items)
    order = np.lexsort((items, dists))                     # primary key D, secondary item
    top = order[:k]
    return items[top], dists[top]


def query(q, s: Snapshot, nprobe: int, k: int):
    """Steps 1-5 for one query.  Returns (ids[k], dist[k], P[nprobe], d_P[nprobe], Dc[nprobe][L])."""
    d = step1_centroid_distances(q, s)
    probes = step2_probe_select(d, nprobe)
    lut = step3_adc_tables(q, s, probes)
    cand = step4_candidate_distances(s, probes, lut)
    items = s.ids[probes].reshape(-1).astype(np.int64)     # flattened S^orig: rank rho, then slot j
    out_ids, out_d = step5_topk(items, cand.reshape(-1), k)
    return out_ids, out_d, probes, d[probes], cand


def query_batch(s: Snapshot, queries, nprobe: int, k: int, rows=None) -> dict:
    """Run `query` for every row (or the given subset `rows`) of `queries`; outputs in the
    C-ABI's layouts: out_ids [Q][k], out_dist [Q][k], trace_lists / trace_list_dist [Q][nprobe],
    trace_cand_dist [Q][nprobe][L] -- int32, distances int64 in the fixed-point variant."""
    queries = np.asarray(queries, dtype=np.int32 if s.fx else np.int8)
    rows = np.arange(queries.shape[0]) if rows is None else np.asarray(rows)
    nq = len(rows)
    dt = np.int64 if s.fx else np.int32
    out = {
        "out_ids": np.empty((nq, k), np.int32),
        "out_dist": np.empty((nq, k), dt),
        "trace_lists": np.empty((nq, nprobe), np.int32),
        "trace_list_dist": np.empty((nq, nprobe), dt),
        "trace_cand_dist": np.empty((nq, nprobe, s.L), dt),
    }
    for a, r in enumerate(rows):
        ids, dd, p, dp, cand = query(queries[r], s, nprobe, k)
        out["out_ids"][a] = ids
        out["out_dist"][a] = dd
        out["trace_lists"][a] = p
        out["trace_list_dist"][a] = dp
        out["trace_cand_dist"][a] = cand
    return out


# ----------------------------------------------------------------------------------------
# Prover witness of one query (§4.7, "Multiset-Based Design")
# ----------------------------------------------------------------------------------------

def witness(q, s: Snapshot, nprobe: int):
    """The witness values the multiset-based prover takes from the off-circuit run of the query
    (PAPER.md:617-618):
      * S^sorted_{idx,dist}: all n_list pairs (i, d_i) sorted, ties by i (R9);
      * the selected LUT entries l^{(m)}_{i,j} = LUT_{i,m,v^{(m)}_{i,j}} for i in P(q), j in [n],
        m in [M], literal Step-3 tables, padding slots included (their code 0);
      * S^sorted_{item,dist}: all N_sel candidate pairs (item, D) sorted, ties by
        item (R10).
    Returns (order[nlist], order_dist[nlist], ell[nprobe][L][M], items[N_sel], dists[N_sel])."""
    d = step1_centroid_distances(q, s)
    order = np.lexsort((np.arange(s.nlist), d))            # primary key d, secondary i
    probes = order[:nprobe]
    lut = step3_adc_tables(q, s, probes)                     # [nprobe][M][Ks]
    m_idx = np.arange(s.M)[None, :]
    ell = np.stack([lut[rho][m_idx, s.codes[i].astype(np.int64)] for rho, i in enumerate(probes)])
    cand = step4_candidate_distances(s, probes, lut)         # [nprobe][L]
    items = s.ids[probes].reshape(-1).astype(np.int64)
    dists = cand.reshape(-1)
    o2 = np.lexsort((items, dists))
    return order, d[order], ell, items[o2], dists[o2]
