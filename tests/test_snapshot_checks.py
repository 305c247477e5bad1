"""The full-size snapshot checker (tests/snapshot_checks.py) accepts the oracle's snapshot and
rejects corrupted ones -- so a GPU snapshot that passes it obeys the build rules."""
import numpy as np
import pytest

import oracle
from synth import generate, get_config

from .snapshot_checks import check_snapshot


@pytest.fixture(scope="module")
def case():
    cfg = get_config("c0")
    inp = generate(cfg)
    s = oracle.build_snapshot(inp.db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, inp.centroid_rows, inp.codeword_rows)
    snap = {"centroids": s.centroids, "codebooks": s.codebooks, "ids": s.ids, "codes": s.codes,
            "counts": s.counts, "list_of": s.list_of}
    return cfg, inp, snap


def test_accepts_oracle_snapshot(case):
    cfg, inp, snap = case
    check_snapshot(cfg, inp, snap, np.random.default_rng(0), n_replay=300, n_slots=300)


def _mutations(snap):
    i = int(np.argmax(snap["counts"]))          # a list with members
    j = int(np.argmin(snap["counts"]))
    yield "swap two members", lambda s: s["ids"][i].__setitem__(slice(0, 2), s["ids"][i][[1, 0]])
    yield "wrong code", lambda s: s["codes"][i, 0].__setitem__(0, (int(s["codes"][i, 0, 0]) + 1) % 16)
    yield "codeword not saturated", lambda s: s["codebooks"][0, 0].__setitem__(0, s["codebooks"][0, 0, 0] ^ 1)
    yield "padding id", lambda s: s["ids"][j].__setitem__(-1, 0)
    yield "centroid", lambda s: s["centroids"][0].__setitem__(0, s["centroids"][0, 0] ^ 1)


@pytest.mark.parametrize("k", range(5))
def test_rejects_corrupted_snapshot(case, k):
    cfg, inp, snap = case
    name, mutate = list(_mutations(snap))[k]
    bad = {key: v.copy() for key, v in snap.items()}
    mutate(bad)
    with pytest.raises(AssertionError):
        check_snapshot(cfg, inp, bad, np.random.default_rng(0), n_replay=300, n_slots=10**6)


def test_rejects_wrong_placement(case):
    """Move one vector to a list ranked after the one the greedy rule picks: the replay fails."""
    cfg, inp, snap = case
    bad = {key: v.copy() for key, v in snap.items()}
    # vector t sits in list a; move it into a list b with room (relabel ids / list_of / counts)
    counts = bad["counts"]
    b = int(np.argmin(counts))
    a = int(np.argmax(counts))
    t = int(bad["ids"][a, counts[a] - 1])
    bad["ids"][a, counts[a] - 1] = -1
    bad["codes"][a, counts[a] - 1] = 0
    counts[a] -= 1
    pos = int(np.searchsorted(bad["ids"][b, :counts[b]], t))
    row = list(bad["ids"][b, :counts[b]])
    row.insert(pos, t)
    bad["ids"][b, :counts[b] + 1] = row
    counts[b] += 1
    bad["list_of"][t] = b
    with pytest.raises(AssertionError):
        check_snapshot(cfg, inp, bad, np.random.default_rng(0), n_replay=inp.db.shape[0], n_slots=10)


@pytest.fixture(scope="module")
def fx_case():
    """The 16-bit fixed-point variant (NEXT-1): C0's float draws encoded by the oracle."""
    from types import SimpleNamespace
    from synth import generate_float
    cfg = get_config("c0")
    f = generate_float(cfg)
    db = oracle.encode_fixed_point(f.db, f.v_max)
    s = oracle.build_snapshot(db, cfg.nlist, cfg.L, cfg.M, cfg.Ks, f.centroid_rows, f.codeword_rows)
    snap = {"centroids": s.centroids, "codebooks": s.codebooks, "ids": s.ids, "codes": s.codes,
            "counts": s.counts, "list_of": s.list_of}
    return cfg, SimpleNamespace(db=db, centroid_rows=f.centroid_rows, codeword_rows=f.codeword_rows), snap


def test_fx_checker_accepts_and_rejects(fx_case):
    cfg, inp, snap = fx_case
    check_snapshot(cfg, inp, snap, np.random.default_rng(0), n_replay=300, n_slots=300, fx=True)
    with pytest.raises(AssertionError):        # the int8 rules (saturated int8 codewords) do not hold
        check_snapshot(cfg, inp, snap, np.random.default_rng(0), n_replay=10, n_slots=10, fx=False)
    bad = {key: v.copy() for key, v in snap.items()}
    m, c, u = np.argwhere(np.abs(bad["codebooks"]) > 127)[0]
    bad["codebooks"][m, c, u] = np.clip(bad["codebooks"][m, c, u], -127, 127)   # R5 applied where R19 binds
    with pytest.raises(AssertionError):
        check_snapshot(cfg, inp, bad, np.random.default_rng(0), n_replay=10, n_slots=10, fx=True)
    bad = {key: v.copy() for key, v in snap.items()}
    i = int(np.argmax(bad["counts"]))
    bad["codes"][i, 0, 0] = (int(bad["codes"][i, 0, 0]) + 1) % cfg.Ks
    with pytest.raises(AssertionError):
        check_snapshot(cfg, inp, bad, np.random.default_rng(0), n_replay=10, n_slots=10**6, fx=True)
