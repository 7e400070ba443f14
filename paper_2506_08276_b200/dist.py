"""Multi-GPU plumbing of the search path (one process per GPU, torch.distributed).

The path shards by query: graph, PQ codes, token store and encoder
weights are replicated on every rank; rank r serves its own slice of each step's
queries; the only collective is the gather of the result ids and scores. NCCL on
GPUs (NVLink/NVSwitch); the same functions run on gloo for CPU tests.
"""
from __future__ import annotations

import numpy as np


def shard_queries(step: int, rank: int, world: int, batch: int, n_queries: int) -> np.ndarray:
    """Indices of the queries rank `rank` serves at `step`: per-rank batches of
    `batch` consecutive queries, ranks interleaved, cycling over the pool (weak
    scaling: per-rank work is fixed as `world` grows)."""
    start = ((step * world + rank) * batch) % n_queries
    return (np.arange(batch, dtype=np.int64) + start) % n_queries


def gather_results(ids, dist_, group=None):
    """All-gather per-rank [batch, k] ids / scores into [world * batch, k] (rank-major)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if world == 1:
        return ids, dist_
    ids = ids.contiguous()
    dist_ = dist_.contiguous()
    if ids.is_cuda and dist.get_backend(group) != "nccl":  # gloo: gather through the host
        gi, gd = gather_results(ids.cpu(), dist_.cpu(), group)
        return gi.to(ids.device), gd.to(dist_.device)
    if ids.is_cuda:
        g_ids = torch.empty((world * ids.shape[0],) + tuple(ids.shape[1:]), dtype=ids.dtype,
                            device=ids.device)
        g_d = torch.empty((world * dist_.shape[0],) + tuple(dist_.shape[1:]), dtype=dist_.dtype,
                          device=dist_.device)
        dist.all_gather_into_tensor(g_ids, ids, group=group)
        dist.all_gather_into_tensor(g_d, dist_, group=group)
        return g_ids, g_d
    li = [torch.empty_like(ids) for _ in range(world)]
    ld = [torch.empty_like(dist_) for _ in range(world)]
    dist.all_gather(li, ids, group=group)
    dist.all_gather(ld, dist_, group=group)
    return torch.cat(li), torch.cat(ld)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """The slowest rank's time (multi-GPU numbers are max over ranks)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    if dist.get_backend(group) != "nccl":
        device = None
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(values, device=None, group=None) -> list:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return [float(v) for v in values]
    if dist.get_backend(group) != "nccl":
        device = None
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    dist.all_reduce(t, group=group)
    return [float(v) for v in t.tolist()]
