"""Multi-GPU plumbing for the nested-Winograd layers (torch.distributed).

The path partitions by batch: every image and every slice is independent, so
ranks share nothing on the data path.  The only collective is one broadcast of
the transformed filter U from rank 0 (NCCL over NVLink on the GPU box, gloo in
the CPU tests), outside any timed region.  Timing is the max over ranks of
each rank's own CUDA-event time.  No compute happens here: the kernels run in
libnw.so through ``conv.NestedConv2d``.
"""
from __future__ import annotations

from typing import Tuple

import torch
import torch.distributed as dist


def world() -> Tuple[int, int]:
    """(rank, world_size); (0, 1) when torch.distributed is not initialised."""
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard(n_total: int, world_size: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced batch shard of rank: (first image, image count).
    The first n_total % world_size ranks take one extra image."""
    if world_size < 1 or not 0 <= rank < world_size or n_total < 0:
        raise ValueError("bad shard request")
    base, extra = divmod(n_total, world_size)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def broadcast_filter(U: torch.Tensor, src: int = 0) -> torch.Tensor:
    """Broadcast the transformed filter (any dtype, viewed as bytes) from src in place."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.broadcast(U, src=src)
    return U


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (e.g. CUDA-event milliseconds) over all ranks."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_batch(y_local: torch.Tensor) -> torch.Tensor:
    """Concatenate every rank's output shard along the batch (verification only; shards may differ in size)."""
    rank, ws = world()
    if ws == 1:
        return y_local
    n = torch.tensor([y_local.shape[0]], dtype=torch.int64, device=y_local.device)
    sizes = [torch.zeros_like(n) for _ in range(ws)]
    dist.all_gather(sizes, n)
    nmax = int(max(s.item() for s in sizes))
    pad = torch.zeros((nmax - y_local.shape[0],) + tuple(y_local.shape[1:]), dtype=y_local.dtype,
                      device=y_local.device)
    buf = torch.cat([y_local, pad]) if pad.numel() else y_local.contiguous()
    out = [torch.empty_like(buf) for _ in range(ws)]
    dist.all_gather(out, buf)
    return torch.cat([o[:int(s.item())] for o, s in zip(out, sizes)])
