"""Multi-GPU plumbing: request sharding and counter aggregation.

Requests are independent, so a batch of N requests is split into
contiguous shards, one per rank (one process per GPU).  Each rank runs the
whole decode loop — controller included — on its shard; nothing crosses GPUs
on the hot path.  Collectives are used only to aggregate statistics after the
timed region: the max of the per-rank device times (the job's wall time) and
the sum of committed tokens.  Backend-agnostic: NCCL on the B200 box, gloo in
the CPU tests.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    start: int      # first global request id of this rank
    count: int      # requests on this rank

    def global_ids(self) -> range:
        return range(self.start, self.start + self.count)


def shard_requests(n_total: int, world: int, rank: int) -> Shard:
    """Contiguous, balanced split (the first n_total % world ranks get one more)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(n_total, world)
    count = base + (1 if rank < extra else 0)
    start = rank * base + min(rank, extra)
    return Shard(rank, world, start, count)


def world_info():
    """(world_size, rank) from torch.distributed when initialised, else (1, 0)."""
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist.get_world_size(), dist.get_rank()
    except Exception:
        pass
    return 1, 0


def aggregate(device_seconds: float, committed_tokens: int, device=None) -> tuple[float, int]:
    """Job-level (max seconds over ranks, total committed tokens)."""
    world, _ = world_info()
    if world == 1:
        return float(device_seconds), int(committed_tokens)
    import torch
    import torch.distributed as dist
    dev = device if device is not None else (
        torch.device("cuda", torch.cuda.current_device())
        if dist.get_backend() == "nccl" else torch.device("cpu"))
    t = torch.tensor([device_seconds], dtype=torch.float64, device=dev)
    n = torch.tensor([committed_tokens], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(n, op=dist.ReduceOp.SUM)
    return float(t.item()), int(n.item())


def gather_objects(obj):
    """All-gather arbitrary per-rank records (e.g. per-shard reports)."""
    world, _ = world_info()
    if world == 1:
        return [obj]
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, obj)
    return out
