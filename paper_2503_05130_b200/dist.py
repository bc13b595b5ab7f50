"""Multi-GPU scenario sharder.

Scenarios are independent, so ranks never communicate inside the slot loop.  Each
rank owns a block of scenarios (its own handle and workspace on its own GPU); the
only collective is one ``all_reduce(SUM)`` of the int64 tally vector at the end of a
step over the NCCL process group (NVLink 5 / NVSwitch; 136 bytes, latency-bound).
int64 sums and the uint64 wrap-sum hash are associative, so the aggregate is
bit-identical for any number of ranks.  Field 16 (max_active) is a sum of
per-scenario maxima by definition.
"""
from __future__ import annotations

import os
from typing import Optional, Tuple

import numpy as np


def env_rank() -> Tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (defaults 0, 1, 0)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def block(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block [lo, hi) of n units owned by rank (sizes differ by at most 1)."""
    return n * rank // world, n * (rank + 1) // world


def init(backend: str = "nccl", device=None):
    """Initialise the default process group when launched with world_size > 1.  With NCCL
    the caller has already selected its GPU (torch.cuda.set_device) and passes it as
    ``device`` (bound to the group: eager communicator init on the right device)."""
    import torch.distributed as dist
    rank, world, _ = env_rank()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        kw = {"device_id": device} if (backend == "nccl" and device is not None) else {}
        dist.init_process_group(backend=backend, rank=rank, world_size=world, **kw)
    return rank, world


def finalize():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()


def allreduce_tallies(t, group=None):
    """In-place SUM all-reduce of an int64 tally tensor (no-op for one rank).  The
    uint64 hash field wraps identically under int64 two's-complement addition."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        if dist.get_backend(group) == "gloo" and t.is_cuda:   # gloo: host copy
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def allreduce_max(x: float) -> float:
    """Max over ranks of a host float (device time of the slowest rank)."""
    import torch
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
        v = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        return float(v.item())
    return x


def barrier():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
