"""Batch sharding across ranks: the method partitions by batch -- every image's
forward is independent given static per-layer scales, the ACU table and the weights are
replicated -- so rank r takes a contiguous slice of the batch and the outputs are collected
with one all-gather at the end (row a8).  Integer results do not depend on the rank count
(A23), which tests/test_multiproc_cpu.py checks with the gloo backend."""
from __future__ import annotations

import torch


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, stop) of `total` items for `rank`; the first total % world ranks
    take one extra item."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gather_rows(local: torch.Tensor, out: torch.Tensor, total: int, dist=None) -> torch.Tensor:
    """Collect every rank's rows of a [total, ...] tensor into `out` on every rank.
    Equal shards use one all_gather_into_tensor (NCCL); uneven shards fall back to a padded
    all-gather.  Without a process group the local rows are copied."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        out.copy_(local)
        return out
    world, rank = dist.get_world_size(), dist.get_rank()
    sizes = [shard_range(total, world, r) for r in range(world)]
    n_max = max(b - a for a, b in sizes)
    if all(b - a == n_max for a, b in sizes) and dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(out, local.contiguous())
        return out
    pad = torch.zeros((n_max,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    for (a, b), part in zip(sizes, parts):
        out[a:b] = part[:b - a]
    return out
