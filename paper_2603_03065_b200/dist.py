"""Host-side plumbing of the multi-GPU path: one process per GPU, each owning a
replica of the snapshot and an independent query batch (the query path partitions by query, so
there is no data-path collective).  torch.distributed is used only for the barrier and the
max-over-ranks of the timings.  Backend-agnostic, so the same code runs under gloo on CPU in the
tests and under NCCL in bench.py."""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def world_from_env() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) as torchrun sets them; (0, 1, 0) when launched plainly."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(world: int, backend: str, device=None) -> None:
    if world > 1 and not dist.is_initialized():
        kw = {"device_id": device} if backend == "nccl" and device is not None else {}
        dist.init_process_group(backend, **kw)


def barrier(world: int) -> None:
    if world > 1:
        dist.barrier()


def max_over_ranks(x: float, world: int, device="cpu") -> float:
    """The job's time is the slowest rank's (weak scaling: every rank does the same work)."""
    if world <= 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def shutdown(world: int) -> None:
    if world > 1 and dist.is_initialized():
        dist.destroy_process_group()
