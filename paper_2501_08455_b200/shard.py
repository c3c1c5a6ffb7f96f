"""Batch sharding across ranks (one process per GPU, torch.distributed).

The signature of a path depends on that path alone (the
reference's rows are bitwise independent, tests/test_kernels.cpp:252-263),
so multi-GPU execution is pure data parallelism: contiguous row blocks per
rank, no collective on the data path. The only communication is (optionally)
gathering the output rows and reducing timings, both host-side plumbing.
"""
from __future__ import annotations


def shard_rows(B: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [lo, hi) of a B-row batch owned by `rank` (contiguous, ceil-split,
    the same split as sigk_signature_sharded_*)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    per = (B + world - 1) // world
    lo = min(B, rank * per)
    return lo, min(B, lo + per)


def gather_rows(local, B: int, group=None):
    """All-gather each rank's (rows, D) shard into the full (B, D) batch on every
    rank (torch tensors; works with gloo on CPU and nccl on GPU)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    per = (B + world - 1) // world
    D = local.shape[1]
    padded = torch.zeros((per, D), dtype=local.dtype, device=local.device)
    padded[: local.shape[0]] = local
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    full = torch.cat(parts, dim=0)
    return full[:B]


def max_over_ranks(x: float, device=None, group=None) -> float:
    """The slowest rank's value (multi-GPU timings are reported as the max)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
