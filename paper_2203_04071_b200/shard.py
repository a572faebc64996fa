"""Batch sharding across ranks: the method partitions by batch -- every image's
forward is independent given static per-layer scales, the ACU table and the weights are
replicated -- so rank r takes a contiguous slice of the batch and the outputs are collected
with one all-gather at the end (row a8).  The paper's analogue is its OpenMP threads "shared
between batches" (§IV.A).  Integer results do not depend on the rank count (A23).

Dynamically calibrated single layers (BJ configs[1], [2]) need one more collective: the
per-tensor max of the WHOLE input (reading A7), so each rank's local amax is all-reduced with
MAX before the scale is formed -- then every rank quantizes with exactly the scale a single
GPU would use and the gathered output equals the G = 1 output bit for bit.

tests/test_multiproc_cpu.py checks this host logic with the gloo backend (world size 2) and
tests/test_gpu_multiproc.py runs two ranks of the device path on one GPU (gloo, host copies).
"""
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


def _active(dist) -> bool:
    return dist is not None and dist.is_initialized() and dist.get_world_size() > 1


def _host_staged(dist, t: torch.Tensor) -> bool:
    """gloo collectives run on host tensors: device tensors are staged through the host."""
    return t.is_cuda and dist.get_backend() != "nccl"


def all_reduce_max_(t: torch.Tensor, dist=None) -> torch.Tensor:
    """In-place MAX all-reduce (e.g. the fp32 amax of a sharded input before axq_scale, so the
    scale equals the single-GPU one).  Exact: max is order-free."""
    if not _active(dist):
        return t
    if _host_staged(dist, t):
        h = t.detach().cpu()
        dist.all_reduce(h, op=dist.ReduceOp.MAX)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t


def gather_rows(local: torch.Tensor, out: torch.Tensor, total: int, dist=None) -> torch.Tensor:
    """Collect every rank's rows of a [total, ...] tensor into `out` on every rank.
    Equal shards on NCCL use one all_gather_into_tensor; uneven shards (or gloo) use a padded
    all-gather, staged through host memory for device tensors on gloo.  Without a process group
    the local rows are copied."""
    if not _active(dist):
        out.copy_(local)
        return out
    world = dist.get_world_size()
    sizes = [shard_range(total, world, r) for r in range(world)]
    n_max = max(b - a for a, b in sizes)
    if all(b - a == n_max for a, b in sizes) and dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(out, local.contiguous())
        return out
    staged = _host_staged(dist, local)
    src = local.detach().cpu() if staged else local
    pad = torch.zeros((n_max,) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
    pad[:src.shape[0]] = src
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    for (a, b), part in zip(sizes, parts):
        out[a:b] = part[:b - a].to(out.device)
    return out


def replica_checksum(tensors, device=None) -> torch.Tensor:
    """A position-weighted int64 checksum of the replicated state (ACU table codes, weight
    codes, static scales as raw bits): two ranks holding different bytes anywhere get different
    sums (up to a 2^-61-ish collision chance).  Returns a 1-element int64 tensor."""
    acc = None
    for i, t in enumerate(tensors):
        t = torch.as_tensor(t)
        if device is not None:
            t = t.to(device)
        b = t.detach().contiguous().reshape(-1).view(torch.uint8).to(torch.int64)
        w = (torch.arange(b.numel(), device=b.device, dtype=torch.int64) % 65521) + 1 + 7919 * i
        s = (b * w).sum().reshape(1)
        acc = s if acc is None else acc * 1000003 + s
    return acc if acc is not None else torch.zeros(1, dtype=torch.int64, device=device)


def verify_replicas(tensors, dist=None, device=None) -> int:
    """Setup-time check that every rank holds identical replicated state ("each
    rank generates them from the seed, and a setup-time checksum all-reduce confirms they are
    identical").  MIN and MAX all-reduces of the checksum must agree; raises otherwise.
    Returns the checksum."""
    c = replica_checksum(tensors, device)
    if not _active(dist):
        return int(c.item())
    lo, hi = c.clone(), c.clone()
    if _host_staged(dist, c):
        lo, hi = lo.cpu(), hi.cpu()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX)
    if int(lo.item()) != int(hi.item()):
        raise RuntimeError("replicated tables / weights differ across ranks (checksums %d .. %d)"
                           % (int(lo.item()), int(hi.item())))
    return int(c.item())
