"""Helpers shared by the GPU parity tests (test infrastructure)."""
from __future__ import annotations

import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np

import oracle

_S = None
_Q = None


def _init(s, q):
    global _S, _Q
    _S, _Q = s, q
    os.environ.setdefault("OMP_NUM_THREADS", "1")


def _work(args):
    rows, nprobe, k = args[:3]
    out = oracle.query_batch(_S, _Q, nprobe, k, rows=rows)
    if len(args) > 3 and not args[3]:       # the candidate trace is not wanted for this shard
        out["trace_cand_dist"] = out["trace_cand_dist"][:0]
    return out


def oracle_queries(s, queries, nprobe, k, rows=None, workers=None):
    """oracle.query_batch over `rows`, sharded over a process pool (fork)."""
    rows = np.arange(queries.shape[0]) if rows is None else np.asarray(rows)
    workers = workers or min(32, len(os.sched_getaffinity(0)))
    if workers <= 1 or len(rows) < 64:
        return oracle.query_batch(s, queries, nprobe, k, rows=rows)
    shards = np.array_split(rows, workers * 4)
    import multiprocessing as mp
    with ProcessPoolExecutor(workers, mp_context=mp.get_context("fork"), initializer=_init,
                             initargs=(s, queries)) as ex:
        parts = list(ex.map(_work, [(sh, nprobe, k) for sh in shards if len(sh)]))
    return {key: np.concatenate([p[key] for p in parts]) for key in parts[0]}


_G = None


def _init_check(s, q, got):
    global _S, _Q, _G
    _S, _Q, _G = s, q, got
    os.environ.setdefault("OMP_NUM_THREADS", "1")


def _check(args):
    pos, rows, nprobe, k = args   # pos: positions of `rows` inside the GPU arrays
    out = oracle.query_batch(_S, _Q, nprobe, k, rows=rows)
    bad = []
    for key, exp in out.items():
        got = _G[key][pos]
        if not np.array_equal(got, exp):
            bad.append(f"{key} rows {int(rows[0])}..{int(rows[-1])}: {first_mismatch(got, exp)}")
    return bad


def oracle_check(s, queries, nprobe, k, got: dict, rows=None, workers=None) -> list:
    """Compare GPU outputs `got` (host arrays whose first axis is `rows`, default every query) with
    oracle.query_batch on s, row by row, in a process pool whose workers compare in place (fork:
    the GPU arrays are shared, nothing large is pickled).  Returns the mismatch descriptions."""
    import multiprocessing as mp
    rows = np.arange(queries.shape[0]) if rows is None else np.asarray(rows)
    workers = workers or min(32, len(os.sched_getaffinity(0)))
    pos = np.arange(len(rows))
    jobs = [(p, rows[p], nprobe, k) for p in np.array_split(pos, max(1, workers * 4)) if len(p)]
    with ProcessPoolExecutor(workers, mp_context=mp.get_context("fork"), initializer=_init_check,
                             initargs=(s, queries, got)) as ex:
        return [b for part in ex.map(_check, jobs) for b in part]


def oracle_queries_all(s, queries, nprobe, k, trace_rows, workers=None):
    """oracle.query_batch over EVERY row of `queries` (process pool); trace_cand_dist is kept only
    for the rows in `trace_rows` (sorted), to bound the host memory and the pickling at C4 sizes.
    Returns (outputs without the trace for all rows, trace_cand_dist for trace_rows)."""
    import multiprocessing as mp
    workers = workers or min(32, len(os.sched_getaffinity(0)))
    rows = np.arange(queries.shape[0])
    shards = [sh for sh in np.array_split(rows, workers * 4) if len(sh)]
    want = set(int(r) for r in trace_rows)
    with ProcessPoolExecutor(workers, mp_context=mp.get_context("fork"), initializer=_init,
                             initargs=(s, queries)) as ex:
        jobs = []
        for sh in shards:   # split every shard into its traced and untraced rows
            tr = np.array([r for r in sh if int(r) in want], dtype=np.int64)
            nt = np.array([r for r in sh if int(r) not in want], dtype=np.int64)
            if len(tr):
                jobs.append((tr, True))
            if len(nt):
                jobs.append((nt, False))
        parts = list(ex.map(_work, [(r, nprobe, k, t) for r, t in jobs]))
    order = np.concatenate([r for r, _ in jobs])
    inv = np.argsort(order)
    full = {key: np.concatenate([p[key] for p in parts])[inv] for key in parts[0] if key != "trace_cand_dist"}
    tr_rows = np.concatenate([r for r, t in jobs if t]) if any(t for _, t in jobs) else np.zeros(0, np.int64)
    tr_vals = np.concatenate([p["trace_cand_dist"] for p, (_, t) in zip(parts, jobs) if t])
    o = np.argsort(tr_rows)
    return full, tr_rows[o], tr_vals[o]


def first_mismatch(a: np.ndarray, b: np.ndarray) -> str:
    if a.shape != b.shape:
        return f"shape {a.shape} vs {b.shape}"
    bad = np.argwhere(a != b)
    if len(bad) == 0:
        return "equal"
    idx = tuple(bad[0])
    return f"{len(bad)} mismatches; first at {idx}: gpu={a[idx]} oracle={b[idx]}"
