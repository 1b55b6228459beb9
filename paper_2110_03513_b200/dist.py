"""Multi-GPU plumbing (host side only): one process per GPU, torch.distributed for the
process group.  Two shardings:

* REPLICATIONS (independent boosting runs that share X): every rank builds the pool
  from the same X and trains its own contiguous block of replications -- no
  collective on the data path.  Collectives are used only for timing (max over
  ranks) and, optionally, to gather results.
* ROWS (include/cwb.h "row sharding"): every rank builds the pool from the full X,
  keeps the row block `row_block(n, rank, world)` and sums s = Zb^T u and r^T r with
  one all-reduce per iteration -- issued by libcwb itself over its own NCCL
  communicator (cwb.Comm(rank, world, unique_id=nccl_unique_id(w))), or through
  torch.distributed (cwb.Comm(rank, world, fn=torch_allreduce_fn())).
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


def gather_results(out: dict, w: World) -> dict:
    """Replication sharding's one collective: every rank's training outputs of its block
    of replications -- offset [B], theta_agg [B, K, d], k/sse/risk traces [M, B] -- packed into one
    [B, 1 + K d + 3 M] float64 tensor and all-gathered in rank order (one NCCL all-gather on the GPU).
    Returns the same keys with the replication axis of all ranks (rank r's block at [r B, (r+1) B))."""
    import torch
    off, agg = out["offset"], out["theta_agg"]
    B, K, d = agg.shape
    tr = [out[k] for k in ("k_trace", "sse_trace", "risk_trace")]
    M = tr[0].shape[0]
    pack = torch.cat([off.reshape(B, 1).to(torch.float64), agg.reshape(B, K * d)] +
                     [t.t().to(torch.float64) for t in tr], 1).contiguous()
    if w.size > 1:
        import torch.distributed as dist
        full = torch.empty((w.size * B, pack.shape[1]), dtype=pack.dtype, device=pack.device)
        dist.all_gather_into_tensor(full, pack)
    else:
        full = pack
    Bt = full.shape[0]
    o = 1 + K * d
    return {"offset": full[:, 0].contiguous(), "theta_agg": full[:, 1:o].reshape(Bt, K, d),
            "k_trace": full[:, o:o + M].t().to(torch.int32).contiguous(),
            "sse_trace": full[:, o + M:o + 2 * M].t().contiguous(),
            "risk_trace": full[:, o + 2 * M:o + 3 * M].t().contiguous()}


def row_block(n: int, rank: int, world: int) -> range:
    """Rows [floor(n r / W), floor(n (r+1) / W)) of rank r: the block libcwb keeps after an
    attach (cwb_rows.cu restrict_rows uses the same formula)."""
    if world < 1 or not 0 <= rank < world or n < world:
        raise ValueError("need 0 <= rank < world <= n")
    return range(n * rank // world, n * (rank + 1) // world)


def broadcast_bytes(data: bytes | None, w: World, src: int = 0, device="cpu") -> bytes:
    """Rank src's bytes on every rank (e.g. the 128-byte NCCL unique id)."""
    if w.size <= 1:
        return bytes(data)
    import torch
    import torch.distributed as dist
    n = torch.tensor([len(data) if w.rank == src else 0], dtype=torch.int64, device=device)
    dist.broadcast(n, src)
    buf = torch.zeros(int(n.item()), dtype=torch.uint8, device=device)
    if w.rank == src:
        buf.copy_(torch.frombuffer(bytearray(data), dtype=torch.uint8))
    dist.broadcast(buf, src)
    return bytes(buf.cpu().numpy().tobytes())


def nccl_unique_id(w: World, device="cpu") -> bytes:
    """A libcwb NCCL unique id made on rank 0 and broadcast to all ranks."""
    from . import cwb
    uid = cwb.cwb_comm_unique_id() if w.rank == 0 else None
    return broadcast_bytes(uid, w, 0, device)


class _DevArray:
    """__cuda_array_interface__ view of a raw device fp64 array (no copy)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 2, "strides": None}


def device_view(ptr: int, count: int, device="cuda"):
    import torch
    return torch.as_tensor(_DevArray(ptr, count), device=device)


def torch_allreduce_fn(device="cuda"):
    """A cwb_comm_init_fn collective over the default torch.distributed group: sums the
    library's device buffer in place.  The library's stream is synchronised first and the
    sum is complete when the callback returns (the stream contract of cwb_allreduce_fn)."""
    import torch
    import torch.distributed as dist

    def fn(ptr, count, stream):
        torch.cuda.synchronize(device)
        t = device_view(ptr, count, device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        torch.cuda.synchronize(device)
    return fn
