"""Multi-GPU plumbing (host side only): one process per GPU, torch.distributed for the
process group.  The hot path shards over REPLICATIONS (independent boosting runs that
share X): every rank builds the pool from the same X and trains its
own contiguous block of replications -- no collective on the data path.  Collectives
are used only for timing (max over ranks) and, optionally, to gather results.
"""
from __future__ import annotations

import os
from dataclasses import dataclass


@dataclass(frozen=True)
class World:
    size: int = 1
    rank: int = 0
    local_rank: int = 0


def world_from_env() -> World:
    """RANK / LOCAL_RANK / WORLD_SIZE as set by torchrun (defaults: single process)."""
    return World(int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
                 int(os.environ.get("LOCAL_RANK", "0")))


def replication_block(b_per_rank: int, rank: int) -> range:
    """Weak scaling: rank r owns global replications [r*B, (r+1)*B)."""
    if b_per_rank < 1 or rank < 0:
        raise ValueError("b_per_rank >= 1 and rank >= 0 required")
    return range(rank * b_per_rank, (rank + 1) * b_per_rank)


def split_replications(b_total: int, size: int, rank: int) -> range:
    """Strong scaling: b_total replications in contiguous blocks, the first b_total % size
    ranks one longer (every replication exactly once)."""
    if size < 1 or not 0 <= rank < size or b_total < 0:
        raise ValueError("bad world / replication count")
    base, rem = divmod(b_total, size)
    start = rank * base + min(rank, rem)
    return range(start, start + base + (1 if rank < rem else 0))


def init_process_group(w: World, backend: str, device=None):
    """Initialise torch.distributed for w.size > 1 (rendezvous from MASTER_ADDR / MASTER_PORT)."""
    if w.size <= 1:
        return None
    import torch.distributed as dist
    if not dist.is_initialized():
        kw = {"backend": backend, "rank": w.rank, "world_size": w.size}
        if device is not None and backend == "nccl":
            kw["device_id"] = device
        dist.init_process_group(**kw)
    return dist


def max_over_ranks(value: float, w: World, device="cpu") -> float:
    """The slowest rank's time: the job's time (timing rule: max over ranks)."""
    if w.size <= 1:
        return float(value)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(w: World) -> None:
    if w.size > 1:
        import torch.distributed as dist
        dist.barrier()


def gather_rows(t, w: World):
    """All-gather equally shaped per-rank tensors along dim 0 (rank order)."""
    if w.size <= 1:
        return t
    import torch
    import torch.distributed as dist
    parts = [torch.empty_like(t) for _ in range(w.size)]
    dist.all_gather(parts, t.contiguous())
    return torch.cat(parts, 0)
