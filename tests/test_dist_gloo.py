"""The multi-GPU (replica) path's host logic on CPU: two ranks over gloo.  Each rank
owns an independent query batch; the only collective is the barrier and the max-over-ranks of the
timings that bench.py reports.  Also: under torchrun the reference arm prints on rank 0 only."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    from paper_2603_03065_b200 import dist as pdist
    from synth import get_config, rank_queries

    r, w, lr = pdist.world_from_env()
    pdist.init(w, "gloo")
    pdist.barrier(w)
    t = pdist.max_over_ranks(1.5 + r, w)          # rank r "took" 1.5 + r ms
    q = rank_queries(get_config("c0"), r)
    pdist.shutdown(w)
    out.put((r, w, lr, t, q.shape, int(q.astype(np.int64).sum())))


def test_two_ranks_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(out.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [x[0] for x in res] == [0, 1] and all(x[1] == 2 and x[2] == x[0] for x in res)
    assert all(x[3] == 2.5 for x in res)                  # max over ranks, seen by every rank
    assert res[0][4] == res[1][4] == (64, 16)              # same batch shape (weak scaling)
    assert res[0][5] != res[1][5]                          # independent query batches


def test_reference_arm_prints_on_rank0_only():
    base = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c0", "--steps", "1",
            "--warmup", "1", "--cpu-sample-seconds", "0.2"]
    for rank in (0, 1):
        env = dict(os.environ, RANK=str(rank), WORLD_SIZE="2", LOCAL_RANK=str(rank))
        p = subprocess.run(base + ["--gpus", "2"], capture_output=True, text=True, env=env, timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        lines = [ln for ln in p.stdout.splitlines() if ln.strip()]
        if rank == 0:
            assert len(lines) == 1
            rec = json.loads(lines[0])
            assert rec["impl"] == "reference" and rec["value"] > 0 and rec["n_gpus"] == 2
        else:
            assert lines == []
