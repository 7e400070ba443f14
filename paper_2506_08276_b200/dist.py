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


def _all_gather_rows(t, group=None):
    """All-gather equal-shaped [rows, ...] tensors into [world * rows, ...] (rank-major)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = t.contiguous()
    if t.is_cuda and dist.get_backend(group) == "nccl":
        out = torch.empty((world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype,
                          device=t.device)
        dist.all_gather_into_tensor(out, t, group=group)
        return out
    host = t.cpu()
    parts = [torch.empty_like(host) for _ in range(world)]
    dist.all_gather(parts, host, group=group)
    return torch.cat(parts).to(t.device)


def shard_bounds(B: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous query shard of rank `rank`: rows [lo, hi) of a B-query batch
    (equal ceil(B / world) shards, the last ones possibly short or empty)."""
    per = -(-B // world)
    lo = min(B, rank * per)
    return lo, min(B, lo + per)


def sharded_search(dev_index, Q, params, source, cache=None, max_inflight: int = 0,
                   group=None):
    """One multi-GPU search step: every rank holds the replicated
    index and the full query batch ``Q`` (CUDA float32 [B, dim]), searches its
    contiguous shard with lv_search_batch, and the shards' ids, scores and
    counters are all-gathered — the only collective. Returns CUDA tensors
    ids [B, k], dist [B, k], counters [B, 4], identical on every rank and
    identical to a single-rank search of the whole batch (per-query results do
    not depend on batching, SURVEY 0 finding 1)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    B, k = Q.shape[0], params.k
    lo, hi = shard_bounds(B, rank, world)
    per = -(-B // world)
    ids = torch.full((per, k), -1, dtype=torch.int64, device=Q.device)
    dst = torch.zeros((per, k), dtype=torch.float32, device=Q.device)
    cnt = torch.zeros((per, 4), dtype=torch.int64, device=Q.device)
    if hi > lo:
        out = dev_index.search_device(Q[lo:hi].contiguous(), params, source, cache=cache,
                                      max_inflight=max_inflight)
        ids[:hi - lo] = out["ids"][:hi - lo]
        dst[:hi - lo] = out["dist"][:hi - lo]
        cnt[:hi - lo] = out["counters"][:hi - lo]
    if world == 1:
        return ids[:B], dst[:B], cnt[:B]
    return (_all_gather_rows(ids, group)[:B], _all_gather_rows(dst, group)[:B],
            _all_gather_rows(cnt, group)[:B])


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
