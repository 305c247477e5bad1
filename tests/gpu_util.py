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
    rows, nprobe, k = args
    return oracle.query_batch(_S, _Q, nprobe, k, rows=rows)


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


def first_mismatch(a: np.ndarray, b: np.ndarray) -> str:
    if a.shape != b.shape:
        return f"shape {a.shape} vs {b.shape}"
    bad = np.argwhere(a != b)
    if len(bad) == 0:
        return "equal"
    idx = tuple(bad[0])
    return f"{len(bad)} mismatches; first at {idx}: gpu={a[idx]} oracle={b[idx]}"
