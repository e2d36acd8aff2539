"""Batch sharding across the GPUs of one node.

Images are independent, so the forward path needs no collective: each rank
convolves its own contiguous slice of the batch with replicated weights.
Collectives appear only outside the timed data path: the max-over-ranks
timing reduction and an optional gather of outputs for verification.
"""

import torch


def shard_range(n: int, rank: int, world: int) -> tuple:
    """[start, stop) of rank's slice of n images; sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Reduce a per-rank duration to the job's (slowest rank) duration."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_batch(local: torch.Tensor, n: int, dist=None) -> torch.Tensor:
    """All-gather uneven batch shards back into the full (n, ...) tensor
    (verification only; never inside a timed region)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return local
    world = dist.get_world_size()
    sizes = [shard_range(n, r, world) for r in range(world)]
    biggest = max(b - a for a, b in sizes)
    pad = torch.zeros((biggest,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([p[: b - a] for p, (a, b) in zip(parts, sizes)], dim=0)
